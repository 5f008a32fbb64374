// generic.cu — the generic item executor (fp32 FMA, any row count <= 128, per-row
// causal mask) and the LSE-merge epilogue.
//
// The generic executor runs ANY work unit of the plan: it is the fp32 debug path
// (tcgen05 has no fp32 kind) and the reference executor the optimised kernels
// are checked against (BLEND_PATH_GENERIC).  Per unit it computes, for each row
// (query token, q head) and the unit's keys K_e (a contiguous range of the
// item's page entries):
//     s = q . k / sqrt(D)  (visible iff key_pos <= row_pos),  online softmax,
//     o = sum softmax(s) v, lse2 = log2-sum-exp2 of s*log2(e)
// exactly the per-partial quantity of the cascade (PAPER §7.2).
//
// The merge epilogue combines a token's partials in ascending key-range order
// (reading #17): L = max lse_i + log sum exp(lse_i - max), O = sum exp(lse_i - L) o_i.
#include <cuda_runtime.h>
#include <math.h>

#include "blend.h"
#include "common.cuh"
#include "ptx.cuh"

namespace blend {

constexpr int GEN_ROWS = 128;
constexpr int GEN_KT = 32;

__device__ __forceinline__ void write_row(const AttnParams& p, const RowInfo& ri, int32_t tgt, const float* o,
                                          float inv_l, float lse2, int lane_stride, int lane) {
  if (tgt == PM_SKIP) return;
  if (tgt == PM_DIRECT) {
    int64_t base = ((int64_t)ri.token * p.hq + ri.head) * p.d;
    for (int e = lane; e < p.d; e += lane_stride) st_elem(p.out, base + e, o[e] * inv_l, p.kv_f32);
    if (lane == 0) p.lse[(int64_t)ri.token * p.hq + ri.head] = lse2 * kLn2;
  } else {
    int64_t base = ((int64_t)tgt * p.hq + ri.head) * p.d;
    for (int e = lane; e < p.d; e += lane_stride) p.ws_o[base + e] = o[e] * inv_l;
    if (lane == 0) p.ws_lse[(int64_t)tgt * p.hq + ri.head] = lse2;
  }
}

// One CTA (128 threads) per unit.  Dynamic smem (fp32):
//   qs[128][D] | os[128][D] | ks[KT][D+1] | vs[KT][D] | ss[128][KT+1] | m,l,alpha[128] | pos[128]
__global__ void __launch_bounds__(128) generic_unit_kernel(AttnParams p) {
  extern __shared__ float sm[];
  const int D = p.d;
  float* qs = sm;
  float* os = qs + GEN_ROWS * D;
  float* ks = os + GEN_ROWS * D;
  float* vs = ks + GEN_KT * (D + 1);
  float* ss = vs + GEN_KT * D;
  float* mrow = ss + GEN_ROWS * (GEN_KT + 1);
  float* lrow = mrow + GEN_ROWS;
  float* arow = lrow + GEN_ROWS;
  int* prow = reinterpret_cast<int*>(arow + GEN_ROWS);

  const Unit u0 = p.units[blockIdx.x];
  // units carry up to 256 rows (two dense tiles): process them 128 rows at a time
  for (int rc = 0; rc < u0.n_rows; rc += GEN_ROWS) {
  Unit u = u0;
  u.row_begin = u0.row_begin + rc;
  u.n_rows = min(GEN_ROWS, u0.n_rows - rc);
  const int nr = u.n_rows;
  const int tid = threadIdx.x;
  __syncthreads();
  for (int idx = tid; idx < nr * D; idx += blockDim.x) {
    int r = idx / D, e = idx % D;
    RowInfo ri = row_info(p, u, r);
    qs[idx] = ld_elem(p.q, ((int64_t)ri.token * p.hq + ri.head) * D + e, p.kv_f32) * p.scale_log2;
    os[idx] = 0.f;
  }
  for (int r = tid; r < nr; r += blockDim.x) {
    RowInfo ri = row_info(p, u, r);
    prow[r] = p.tok_pos[ri.token];
    mrow[r] = -INFINITY;
    lrow[r] = 0.f;
  }
  __syncthreads();

  for (int ei = u.entry_begin; ei < u.entry_end; ++ei) {
    const KvEntry en = p.entries[ei];
    const int64_t kvbase = (((int64_t)en.page * p.hkv + u.kvh) * p.ps + en.row_off) * D;
    for (int k0 = 0; k0 < en.count; k0 += GEN_KT) {
      const int kt = min(GEN_KT, en.count - k0);
      for (int idx = tid; idx < kt * D; idx += blockDim.x) {
        int i = idx / D, e = idx % D;
        ks[i * (D + 1) + e] = ld_elem(p.k_cache, kvbase + (int64_t)(k0 + i) * D + e, p.kv_f32);
        vs[i * D + e] = ld_elem(p.v_cache, kvbase + (int64_t)(k0 + i) * D + e, p.kv_f32);
      }
      __syncthreads();
      for (int idx = tid; idx < nr * kt; idx += blockDim.x) {
        int r = idx / kt, i = idx % kt;
        float s = 0.f;
        const float* qr = qs + r * D;
        const float* kr = ks + i * (D + 1);
        for (int e = 0; e < D; ++e) s = fmaf(qr[e], kr[e], s);
        ss[r * (GEN_KT + 1) + i] = (en.pos0 + k0 + i <= prow[r]) ? s : -INFINITY;
      }
      __syncthreads();
      for (int r = tid; r < nr; r += blockDim.x) {
        float* sr = ss + r * (GEN_KT + 1);
        float mx = mrow[r];
        for (int i = 0; i < kt; ++i) mx = fmaxf(mx, sr[i]);
        float alpha = 1.f, sum = 0.f;
        if (mx == -INFINITY) {
          for (int i = 0; i < kt; ++i) sr[i] = 0.f;
        } else {
          alpha = exp2f(mrow[r] - mx);   // m = -inf -> 0
          for (int i = 0; i < kt; ++i) {
            float pv = exp2f(sr[i] - mx);
            sr[i] = pv;
            sum += pv;
          }
        }
        lrow[r] = lrow[r] * alpha + sum;
        mrow[r] = mx;
        arow[r] = alpha;
      }
      __syncthreads();
      for (int idx = tid; idx < nr * D; idx += blockDim.x) {
        int r = idx / D, e = idx % D;
        const float* sr = ss + r * (GEN_KT + 1);
        float o = os[idx] * arow[r];
        for (int i = 0; i < kt; ++i) o = fmaf(sr[i], vs[i * D + e], o);
        os[idx] = o;
      }
      __syncthreads();
    }
  }
  // finalise: one warp per row
  const int warp = tid >> 5, lane = tid & 31;
  for (int r = warp; r < nr; r += blockDim.x / 32) {
    RowInfo ri = row_info(p, u, r);
    int32_t tgt = row_target(p, u, ri.tl);
    float l = lrow[r];
    float lse2 = l > 0.f ? mrow[r] + log2f(l) : -INFINITY;
    float inv = l > 0.f ? 1.f / l : 0.f;
    write_row(p, ri, tgt, os + r * D, inv, lse2, 32, lane);
  }
  }
}

// One warp per (merged token, 2 q heads); lanes own D/32 contiguous elements.
__global__ void __launch_bounds__(256, 4) merge_kernel(AttnParams p) {   // 4 blocks/SM: one wave at C2
  ptx::pdl_wait();   // launched as a programmatic dependent of the streaming pass
  if (p.trace != nullptr && threadIdx.x == 0) {   // diagnostics: first start / last end
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(p.trace + 296 * 64, t);
  }
  const int h0 = (blockIdx.y * 8 + (threadIdx.x >> 5)) * 2;   // two q heads per warp
  if (h0 < p.hq) warp_merge_heads<2>(p, blockIdx.x, h0, threadIdx.x & 31);
  if (p.trace != nullptr && (threadIdx.x & 31) == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(p.trace + 296 * 64 + 1, t);
  }
}

cudaError_t set_smem_once(const void* func, size_t bytes);

size_t generic_smem_bytes(int D) {
  return sizeof(float) * ((size_t)GEN_ROWS * D * 2 + GEN_KT * (D + 1) + GEN_KT * D + GEN_ROWS * (GEN_KT + 1) +
                          4 * GEN_ROWS);
}

cudaError_t launch_generic(const AttnParams& p, cudaStream_t st) {
  if (p.n_units <= 0) return cudaSuccess;
  size_t smem = generic_smem_bytes(p.d);
  cudaError_t e = set_smem_once((const void*)generic_unit_kernel, smem);
  if (e != cudaSuccess) return e;
  generic_unit_kernel<<<p.n_units, 128, smem, st>>>(p);
  return cudaPeekAtLastError();
}

cudaError_t launch_merge(const AttnParams& p, cudaStream_t st, bool pdl) {
  if (p.n_merge <= 0) return cudaSuccess;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.n_merge, (p.hq + 15) / 16);   // 8 warps x 2 heads per block
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, merge_kernel, p);
}

}  // namespace blend
