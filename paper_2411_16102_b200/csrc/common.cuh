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
  const int32_t* merge_rows;
  int32_t n_units;
  int32_t n_merge;
  int32_t hq, hkv, g, d, ps;
  int32_t kv_f32;   // 1: fp32 q/k/v/out, 0: bf16
  float scale_log2; // log2(e) / sqrt(D)
  int32_t avg_entries;   // host-side launch heuristic: mean entries per unit
  const RowDesc* srows;  // streaming units' row descriptors (SEC_STREAM_ROWS)
  int32_t* sched;        // workspace word: dynamic unit counter of the streaming pass (zeroed per call)
  const int32_t* prow_list;   // partial row -> {merge list, source count} (SEC_PROW_LIST)
  int32_t* arrive;       // arrival counters [partial row][Hq] (workspace; NULL: the merge kernel merges)
  const int32_t* dqtok;  // dense units: first token when the unit's tokens are consecutive, else -1
  int32_t n_tokens;      // query tokens (rows of q / out)
  int32_t dense_ctas;    // dense grid cap from the planner (0: one CTA per SM)
  int32_t merge_nsrc;    // > 0: every unfused merge list has this many sources
  unsigned long long* trace;   // diagnostics only (blend_internal_set_trace): [CTA][64] globaltimer stamps
};

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

// Fused LSE merge (reading #17, ascending key start): this unit's own normalised
// result (o_self[k] for elements e0 + k*stride, lse2_self) is combined with the
// already-written partials of merge list m (entry -1 = self) and stored to out/lse.
__device__ __forceinline__ void fused_merge_store(const AttnParams& p, int32_t tgt, int token, int head,
                                                  const float* o_self, float lse2_self, int e0, int stride, int n,
                                                  bool write_lse) {
  const int m = PM_FUSED_BASE - tgt;
  const int s0 = p.merge_off[m], s1 = p.merge_off[m + 1];
  float M = -INFINITY;
  for (int s = s0; s < s1; ++s) {
    const int32_t row = p.merge_rows[s];
    M = fmaxf(M, row < 0 ? lse2_self : p.ws_lse[(int64_t)row * p.hq + head]);
  }
  float acc[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = 0.f;
  float tot = 0.f;
  if (M != -INFINITY) {
    for (int s = s0; s < s1; ++s) {
      const int32_t row = p.merge_rows[s];
      const float w = exp2f((row < 0 ? lse2_self : p.ws_lse[(int64_t)row * p.hq + head]) - M);
      tot += w;
      const float* src = p.ws_o + ((int64_t)row * p.hq + head) * p.d;
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (k < n) acc[k] = fmaf(w, row < 0 ? o_self[k] : src[e0 + k * stride], acc[k]);
    }
  }
  const float inv = tot > 0.f ? 1.f / tot : 0.f;
  const int64_t ob = ((int64_t)token * p.hq + head) * p.d;
#pragma unroll
  for (int k = 0; k < 16; ++k)
    if (k < n) st_elem(p.out, ob + e0 + k * stride, acc[k] * inv, p.kv_f32);
  if (write_lse) p.lse[(int64_t)token * p.hq + head] = M != -INFINITY ? (M + log2f(tot)) * kLn2 : -INFINITY;
}

// LSE merge of (unfused) merge list m, q head h by one warp (reading #17: the list's
// fixed ascending key-start order, so the result does not depend on who merges or when);
// entry s of an unfused list is partial row s (host planner invariant), so the only
// dependent loads are merge_off -> partials;
// lanes own D/32 contiguous elements.  Partials are read through L2 (ld.global.cg):
// with arrival merging they were written by other SMs during this launch.
template <int NH>
__device__ __forceinline__ void warp_merge_heads(const AttnParams& p, int m, int h0, int lane) {
  // NH q heads of merge list m per warp: both heads' loads of a chunk are in flight
  // together (half the warps of one head per warp, so the grid fits one wave).  32-bit
  // index math, MUFU ex2 / lg2 / rcp, and one vector store per lane and head.
  const int token = p.merge_tok[m];
  // every unfused list of the plan has merge_nsrc sources (e.g. one dense + one streaming
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
        const int r = (ok ? c0 + i : c0) * hq + h;   // unfused: entry s is partial row s
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

// Arrival merging ("the last producer merges", replaces the merge launch).  A producer
// that has written its partial (o, lse) rows and fenced them counts each row in on the
// counter of its list (first partial row, q head); the last of the list's nsrc
// sources merges it.  The counter is left at 0 for the next call (workspace counters
// start zeroed).
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ bool arrive_last(const AttnParams& p, int32_t first, int32_t h, int32_t nsrc) {
  int32_t* c = p.arrive + (int64_t)first * p.hq + h;
  const bool last = atomicAdd(c, 1) == nsrc - 1;
  if (last) {
    *c = 0;
    fence_acq_rel_gpu();   // acquire side: the other sources' partials are read after this
  }
  return last;
}

// Four lanes (sub = 0..3, D/4 contiguous elements each) merge one (token, q head): the
// list's partial rows first .. first + nsrc - 1 in their fixed ascending key-start
// order (reading #17), so the result does not depend on which producer merges.  Out
// row qrow = token * Hq + head (bf16), lse in natural log.  Partials are read through
// L2 (ld.global.cg): other SMs wrote them during this launch.
template <int D>
__device__ __forceinline__ void merge_row4(const AttnParams& p, int first, int nsrc, int h, int qrow, int sub) {
  constexpr int E = D / 4;
  // one online pass over the sources, two at a time: both sources' lse and o loads are
  // in flight together (one memory round trip per pair), then a rescale-accumulate
  float mx = -INFINITY, tot = 0.f;
  float acc[E];
#pragma unroll
  for (int k = 0; k < E; ++k) acc[k] = 0.f;
  for (int i = 0; i < nsrc; i += 2) {
    const bool two = i + 1 < nsrc;
    const int64_t r0 = (int64_t)(first + i) * p.hq + h, r1 = two ? r0 + p.hq : r0;
    const float l0 = __ldcg(p.ws_lse + r0), l1 = two ? __ldcg(p.ws_lse + r1) : -INFINITY;
    float4 v0[E / 4], v1[E / 4];
    const float4* s0 = reinterpret_cast<const float4*>(p.ws_o + r0 * D + sub * E);
    const float4* s1 = reinterpret_cast<const float4*>(p.ws_o + r1 * D + sub * E);
#pragma unroll
    for (int k = 0; k < E / 4; ++k) {
      v0[k] = __ldcg(s0 + k);
      v1[k] = __ldcg(s1 + k);
    }
    const float cm = fmaxf(mx, fmaxf(l0, l1));
    if (cm == -INFINITY) continue;                  // both empty so far
    const float a = exp2f(mx - cm), w0 = exp2f(l0 - cm), w1 = exp2f(l1 - cm);   // -inf -> 0
    tot = tot * a + w0 + w1;
#pragma unroll
    for (int k = 0; k < E / 4; ++k) {
      acc[4 * k] = fmaf(w1, v1[k].x, fmaf(w0, v0[k].x, acc[4 * k] * a));
      acc[4 * k + 1] = fmaf(w1, v1[k].y, fmaf(w0, v0[k].y, acc[4 * k + 1] * a));
      acc[4 * k + 2] = fmaf(w1, v1[k].z, fmaf(w0, v0[k].z, acc[4 * k + 2] * a));
      acc[4 * k + 3] = fmaf(w1, v1[k].w, fmaf(w0, v0[k].w, acc[4 * k + 3] * a));
    }
    mx = cm;
  }
  const float inv = tot > 0.f ? 1.f / tot : 0.f;
  if (p.kv_f32) {
    float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) + (int64_t)qrow * D + sub * E);
#pragma unroll
    for (int k = 0; k < E / 4; ++k)
      dst[k] = make_float4(acc[4 * k] * inv, acc[4 * k + 1] * inv, acc[4 * k + 2] * inv, acc[4 * k + 3] * inv);
  } else {
    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.out) + (int64_t)qrow * D + sub * E);
#pragma unroll
    for (int k = 0; k < E / 8; ++k) {
      uint4 w4;
      __nv_bfloat162 b;
      b = __floats2bfloat162_rn(acc[8 * k] * inv, acc[8 * k + 1] * inv);
      w4.x = *reinterpret_cast<uint32_t*>(&b);
      b = __floats2bfloat162_rn(acc[8 * k + 2] * inv, acc[8 * k + 3] * inv);
      w4.y = *reinterpret_cast<uint32_t*>(&b);
      b = __floats2bfloat162_rn(acc[8 * k + 4] * inv, acc[8 * k + 5] * inv);
      w4.z = *reinterpret_cast<uint32_t*>(&b);
      b = __floats2bfloat162_rn(acc[8 * k + 6] * inv, acc[8 * k + 7] * inv);
      w4.w = *reinterpret_cast<uint32_t*>(&b);
      dst[k] = w4;
    }
  }
  if (sub == 0) p.lse[qrow] = mx != -INFINITY ? (mx + log2f(tot)) * kLn2 : -INFINITY;
}

}  // namespace blend
