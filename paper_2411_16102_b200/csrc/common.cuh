// common.cuh — device helpers shared by libblend's kernels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"
#include "ptx.cuh"

namespace blend {

constexpr float kLn2 = 0.6931471805599453f;
constexpr float kLog2e = 1.4426950408889634f;

// Pointers + dims every attention kernel needs (passed by value).
struct AttnParams {
  const void* q;
  const void* k_cache;
  const void* v_cache;
  void* out;
  float* lse;
  float* ws_o;      // [partial rows][Hq][D] fp32
  float* ws_lse;    // [partial rows][Hq]    fp32, log2 domain
  const int32_t* tok_pos;
  const int32_t* item_tokens;
  const KvEntry* entries;
  const Unit* units;
  const int32_t* partmap;
  const int32_t* merge_tok;
  const int32_t* merge_off;
  int32_t n_units;
  int32_t n_merge;
  int32_t hq, hkv, g, d, ps;
  int32_t kv_f32;   // 1: fp32 q/k/v/out, 0: bf16
  float scale_log2; // log2(e) / sqrt(D)
  int32_t avg_entries;   // host-side launch heuristic: mean entries per unit
  const RowDesc* srows;  // streaming units' row descriptors (SEC_STREAM_ROWS)
  int32_t* sched;        // workspace word: dynamic unit counter of the streaming pass (zeroed per call)
  const int32_t* dqtok;  // dense units: first token when the unit's tokens are consecutive, else -1
  int32_t n_tokens;      // query tokens (rows of q / out)
  int32_t dense_ctas;    // dense grid cap from the planner (0: one CTA per SM)
  int32_t merge_nsrc;    // > 0: every merge list has this many sources
  unsigned long long* trace;   // diagnostics only (blend_internal_set_trace): [CTA][64] globaltimer stamps
  unsigned long long* stats;   // diagnostics only (blend_internal_set_stats): softmax path counters
                               // [STAT_*], NULL in production calls
};

// Softmax path counters (tests assert that peaked inputs drive every rescale path).
enum {
  STAT_DENSE_BLOCKS = 0,     // dense pass: (tile, 64-key block) steps of non-padding warps
  STAT_DENSE_SLOW = 1,       //   ... that took the max-first path (first block of a unit, or a
                             //   fast-path block whose exponentials summed to > 2^8)
  STAT_DENSE_SLOW_LATE = 2,  //   ... of those, slow blocks after a unit's first block
  STAT_DENSE_RESCALE = 3,    //   ... that rescaled O in TMEM (running max grew by > 2^8)
  STAT_STREAM_STAGES = 4,    // streaming pass: 32-key stages
  STAT_STREAM_RESCALE = 5,   //   ... where some row's running max grew (alpha < 1 on a live row)
  STAT_TAIL_ZEROED = 6,      // stages / blocks whose V rows past an entry's count were zeroed
  STAT_COUNT = 8
};
__device__ __forceinline__ void stat_add(const AttnParams& p, int k, unsigned long long v) {
  if (p.stats != nullptr) atomicAdd(p.stats + k, v);
}

// Diagnostics: stamp slot k of this CTA's trace row (no-op unless a trace buffer is set).
__device__ __forceinline__ void trace_stamp(const AttnParams& p, int k) {
  if (p.trace != nullptr && k < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[(size_t)blockIdx.x * 64 + k] = t;
  }
}
// streaming-pass diagnostics: the second half of the trace buffer ([148 + CTA][64])
__device__ __forceinline__ void trace_stamp_s(const AttnParams& p, int k) {
  if (p.trace != nullptr && k < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[(size_t)(148 + blockIdx.x) * 64 + k] = t;
  }
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ float grid_val(uint64_t z) { return (float)((int)(z >> 56) - 128) * (1.0f / 128.0f); }

__device__ __forceinline__ float ld_elem(const void* base, int64_t idx, int f32) {
  return f32 ? __ldg(reinterpret_cast<const float*>(base) + idx)
             : __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[idx]);
}

__device__ __forceinline__ void st_elem(void* base, int64_t idx, float v, int f32) {
  if (f32) reinterpret_cast<float*>(base)[idx] = v;
  else reinterpret_cast<__nv_bfloat16*>(base)[idx] = __float2bfloat16_rn(v);
}

// Row metadata of unit row r: global token, q head, token_local
struct RowInfo {
  int32_t token, head, tl;
};
__device__ __forceinline__ RowInfo row_info(const AttnParams& p, const Unit& u, int r) {
  int ir = u.row_begin + r;
  int tl = ir / p.g;
  RowInfo ri;
  ri.tl = tl;
  ri.token = p.item_tokens[u.tok_base + tl];
  ri.head = u.kvh * p.g + (ir - tl * p.g);
  return ri;
}

// Write one finished row: O already normalised, lse2 in log2 units (-inf if empty).
// DIRECT -> out/lse (natural log); partial row -> workspace; SKIP -> nothing.
__device__ __forceinline__ int32_t row_target(const AttnParams& p, const Unit& u, int tl) {
  return p.partmap[u.pm_base + tl];
}

// LSE merge of merge list m, q head h by one warp (reading #17: the list's
// fixed ascending key-start order, so the result does not depend on who merges or when);
// entry s of a list is partial row s (host planner invariant), so the only dependent
// loads are merge_off -> partials; lanes own D/32 contiguous elements.
template <int NH>
__device__ __forceinline__ void warp_merge_heads(const AttnParams& p, int m, int h0, int lane) {
  // NH q heads of merge list m per warp: both heads' loads of a chunk are in flight
  // together (half the warps of one head per warp, so the grid fits one wave).  32-bit
  // index math, MUFU ex2 / lg2 / rcp, and one vector store per lane and head.
  const int token = p.merge_tok[m];
  // every list of the plan has merge_nsrc sources (e.g. one dense + one streaming
  // partial per decode token): list m is rows m*n .. m*n+n-1, no merge_off round trip
  const int s0 = p.merge_nsrc > 0 ? m * p.merge_nsrc : p.merge_off[m];
  const int s1 = p.merge_nsrc > 0 ? s0 + p.merge_nsrc : p.merge_off[m + 1];
  const int D = p.d, hq = p.hq;
  const int vec = D / 32;          // 2 or 4 elements per lane
  const int e0 = lane * vec;
  constexpr int MCH = 2;
  float mx[NH], tot[NH], acc[NH][4];
#pragma unroll
  for (int j = 0; j < NH; ++j) {
    mx[j] = -INFINITY;
    tot[j] = 0.f;
    acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
  }
  for (int c0 = s0; c0 < s1; c0 += MCH) {
    float l[NH][MCH];
    float4 v[NH][MCH];
#pragma unroll
    for (int j = 0; j < NH; ++j) {
      const int h = h0 + j < hq ? h0 + j : h0;
#pragma unroll
      for (int i = 0; i < MCH; ++i) {
        const bool ok = c0 + i < s1;
        const int r = (ok ? c0 + i : c0) * hq + h;   // entry s is partial row s
        l[j][i] = ok ? __ldcg(p.ws_lse + r) : -INFINITY;
        const float* src = p.ws_o + (size_t)r * D + e0;
        if (vec == 4) {
          v[j][i] = __ldcg(reinterpret_cast<const float4*>(src));
        } else {
          const float2 t = __ldcg(reinterpret_cast<const float2*>(src));
          v[j][i] = make_float4(t.x, t.y, 0.f, 0.f);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < NH; ++j) {
      float cm = mx[j];
#pragma unroll
      for (int i = 0; i < MCH; ++i) cm = fmaxf(cm, l[j][i]);
      if (cm == -INFINITY) continue;
      const float a = ptx::ex2(mx[j] - cm);      // mx = -inf on the first live chunk -> 0
      tot[j] *= a;
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[j][k] *= a;
#pragma unroll
      for (int i = 0; i < MCH; ++i) {
        const float w = ptx::ex2(l[j][i] - cm);  // l = -inf (absent source) -> 0
        tot[j] += w;
        acc[j][0] = fmaf(w, v[j][i].x, acc[j][0]);
        acc[j][1] = fmaf(w, v[j][i].y, acc[j][1]);
        acc[j][2] = fmaf(w, v[j][i].z, acc[j][2]);
        acc[j][3] = fmaf(w, v[j][i].w, acc[j][3]);
      }
      mx[j] = cm;
    }
  }
#pragma unroll
  for (int j = 0; j < NH; ++j) {
    const int h = h0 + j;
    if (h >= hq) break;
    const float inv = tot[j] > 0.f ? ptx::rcp(tot[j]) : 0.f;
    const int64_t ob = (int64_t)(token * hq + h) * D + e0;   // out can exceed 2^31 elements (C4)
    if (p.kv_f32) {
      float* dst = reinterpret_cast<float*>(p.out) + ob;
      if (vec == 4)
        *reinterpret_cast<float4*>(dst) = make_float4(acc[j][0] * inv, acc[j][1] * inv, acc[j][2] * inv, acc[j][3] * inv);
      else
        *reinterpret_cast<float2*>(dst) = make_float2(acc[j][0] * inv, acc[j][1] * inv);
    } else {
      __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.out) + ob;
      const uint32_t b01 = ptx::pack_bf16(acc[j][0] * inv, acc[j][1] * inv);
      if (vec == 4)
        *reinterpret_cast<uint2*>(dst) = make_uint2(b01, ptx::pack_bf16(acc[j][2] * inv, acc[j][3] * inv));
      else
        *reinterpret_cast<uint32_t*>(dst) = b01;
    }
    if (lane == 0) p.lse[token * hq + h] = mx[j] != -INFINITY ? (mx[j] + ptx::lg2(tot[j])) * kLn2 : -INFINITY;
  }
}

}  // namespace blend
