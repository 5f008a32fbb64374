// dense.cu — the dense pass on the 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// Work units with many rows per kv head — a SEPARATE shared-prefix node attended
// once by all the SMALL requests under it (PAPER §5 P:11 "exactly-once computation
// of shared prefixes"; §7.2 P:248-251 cascade reuse of the shared KV access), or a
// BIG request (chunked prefill) — are dense contractions: 128 query rows
// (tokens x grouped q heads) against 128-key blocks of the node's pages.
//
// One persistent CTA per SM, warp-specialised:
//   warp 0      TMA producer: K/V page entries (128B swizzle) -> 2-stage smem ring
//   warp 1      MMA issuer (one thread): S = Q K^T (UMMA 128x128x16, K-major A/B)
//               into a double-buffered TMEM S; O += P V (P K-major from smem, V
//               MN-major) into TMEM O; tcgen05.commit -> mbarriers
//   warp 2      TMEM allocator (512 columns: S0 | S1 | O)
//   warps 4..7  softmax / epilogue: thread = query row = TMEM lane.  tcgen05.ld the
//               S row, per-row causal mask, log2-domain online softmax with lazy
//               O rescaling (only when the running max grows by > 8), P -> bf16
//               smem (128B swizzle), final O / l -> bf16 row or fp32 partial.
// QK_{j+1} runs on the tensor pipe while the softmax of block j runs.
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>

#include "blend.h"
#include "common.cuh"
#include "ptx.cuh"

namespace blend {

constexpr int DN_THREADS = 256;
constexpr int DN_KB = 128;               // keys per block (UMMA N of QK^T, K of PV)
constexpr int DN_CHUNK = 128 * 128;      // 128 rows x 128 B (one 64-column chunk)
constexpr uint32_t DN_TMEM_COLS = 512;
constexpr float DN_RESCALE_T = 8.0f;     // lazy-rescale threshold (log2 units)

struct DenseSmem {
  uint32_t q, p, stage0, stage_stride, bar, total;
  int nstage;
};

__host__ __device__ inline DenseSmem dense_layout(int D) {
  DenseSmem L;
  const int CH = D / 64;
  L.q = 0;
  L.p = CH * DN_CHUNK;
  L.stage0 = L.p + 2 * DN_CHUNK;
  L.stage_stride = 2 * CH * DN_CHUNK;
  L.nstage = D == 128 ? 2 : 4;
  L.bar = L.stage0 + L.nstage * L.stage_stride;
  L.total = L.bar + 256;
  return L;
}

template <int D, int BOX>
__global__ void __launch_bounds__(DN_THREADS, 1)
    dense_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv, AttnParams p) {
  constexpr int CH = D / 64;
  constexpr int EPB = DN_KB / BOX;      // page entries per 128-key block
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const DenseSmem L = dense_layout(D);
  const int NS = L.nstage;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar);
  uint64_t* kv_full = bars;            // [NS]
  uint64_t* kv_empty = bars + 4;       // [NS]
  uint64_t* s_full = bars + 8;         // [2]
  uint64_t* q_full = bars + 10;
  uint64_t* q_empty = bars + 11;
  uint64_t* p_full = bars + 12;
  uint64_t* o_done = bars + 13;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      ptx::mbar_init(&kv_empty[s], 1);
    }
    ptx::mbar_init(&s_full[0], 1);
    ptx::mbar_init(&s_full[1], 1);
    ptx::mbar_init(q_full, 4);
    ptx::mbar_init(q_empty, 1);
    ptx::mbar_init(p_full, 4);
    ptx::mbar_init(o_done, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, DN_TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tmk);
      ptx::tma_prefetch_desc(&tmv);
      uint32_t kit = 0;
      for (int ui = blockIdx.x; ui < p.n_units; ui += gridDim.x) {
        const Unit u = p.units[ui];
        const int ne = u.entry_end - u.entry_begin;
        const int nb = (ne + EPB - 1) / EPB;
        for (int j = 0; j < nb; ++j, ++kit) {
          const uint32_t s = kit % NS, ph = (kit / NS) & 1;
          ptx::mbar_wait(&kv_empty[s], ph ^ 1);
          uint8_t* kst = smem + L.stage0 + s * L.stage_stride;
          uint8_t* vst = kst + CH * DN_CHUNK;
          ptx::mbar_arrive_expect_tx(&kv_full[s], 2u * CH * DN_CHUNK);
#pragma unroll
          for (int i = 0; i < EPB; ++i) {
            int e = u.entry_begin + j * EPB + i;
            if (e >= u.entry_end) e = u.entry_begin;   // pad the last block (masked)
            const KvEntry en = p.entries[e];
            const int32_t y = (en.page * p.hkv + u.kvh) * p.ps + en.row_off;
#pragma unroll
            for (int c = 0; c < CH; ++c) {
              ptx::tma_load_2d(kst + c * DN_CHUNK + i * BOX * 128, &tmk, &kv_full[s], c * 64, y);
              ptx::tma_load_2d(vst + c * DN_CHUNK + i * BOX * 128, &tmv, &kv_full[s], c * 64, y);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      constexpr uint32_t IDESC_QK = ptx::umma_idesc_bf16(128, DN_KB, 0, 0);
      constexpr uint32_t IDESC_PV = ptx::umma_idesc_bf16(128, D, 0, 1);
      const uint32_t q_addr = ptx::smem_u32(smem + L.q);
      const uint32_t p_addr = ptx::smem_u32(smem + L.p);
      uint32_t kit = 0, gb = 0, gu = 0;
      for (int ui = blockIdx.x; ui < p.n_units; ui += gridDim.x) {
        const Unit u = p.units[ui];
        const int nb = (u.entry_end - u.entry_begin + EPB - 1) / EPB;
        ptx::mbar_wait(q_full, gu & 1);
        ptx::tc_fence_after();
        for (int j = 0; j <= nb; ++j) {
          if (j < nb) {
            const uint32_t s = (kit + j) % NS;
            ptx::mbar_wait(&kv_full[s], ((kit + j) / NS) & 1);
            ptx::tc_fence_after();
            const uint32_t kst = ptx::smem_u32(smem + L.stage0 + s * L.stage_stride);
            const uint32_t sb = (gb + j) & 1;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint32_t off = (kk / 4) * DN_CHUNK + (kk % 4) * 32;
              ptx::umma_f16(tmem + sb * DN_KB, ptx::umma_desc_sw128(q_addr + off, 16, 1024),
                            ptx::umma_desc_sw128(kst + off, 16, 1024), IDESC_QK, kk > 0);
            }
            ptx::umma_commit(&s_full[sb]);
            if (j == nb - 1) ptx::umma_commit(q_empty);
          }
          if (j >= 1) {
            const int jj = j - 1;
            const uint32_t s = (kit + jj) % NS;
            ptx::mbar_wait(p_full, (gb + jj) & 1);
            ptx::tc_fence_after();
            const uint32_t vst = ptx::smem_u32(smem + L.stage0 + s * L.stage_stride) + CH * DN_CHUNK;
#pragma unroll
            for (int kk = 0; kk < DN_KB / 16; ++kk) {
              const uint32_t aoff = (kk / 4) * DN_CHUNK + (kk % 4) * 32;
              ptx::umma_f16(tmem + 2 * DN_KB, ptx::umma_desc_sw128(p_addr + aoff, 16, 1024),
                            ptx::umma_desc_sw128(vst + kk * 16 * 128, DN_CHUNK, 1024), IDESC_PV,
                            (jj > 0 || kk > 0) ? 1u : 0u);
            }
            ptx::umma_commit(&kv_empty[s]);
            ptx::umma_commit(o_done);
          }
        }
        kit += nb;
        gb += nb;
        ++gu;
      }
    }
  } else if (warp >= 4) {
    // ===================== softmax / epilogue =====================
    const int r = threadIdx.x - 128;                 // query row = TMEM lane
    const uint32_t lane_base = (uint32_t)((warp - 4) * 32) << 16;
    uint8_t* qs = smem + L.q;
    uint8_t* ps_ = smem + L.p;
    uint32_t gb = 0, gu = 0;
    for (int ui = blockIdx.x; ui < p.n_units; ui += gridDim.x) {
      const Unit u = p.units[ui];
      const int nb = (u.entry_end - u.entry_begin + EPB - 1) / EPB;
      int32_t pos = INT32_MIN, token = 0, head = 0, tgt = PM_SKIP;
      if (r < u.n_rows) {
        RowInfo ri = row_info(p, u, r);
        pos = p.tok_pos[ri.token];
        token = ri.token;
        head = ri.head;
        tgt = row_target(p, u, ri.tl);
      }
      // ---- Q row -> smem (K-major, 128B swizzle); wait until the previous unit's QKs are done
      if (gu > 0) ptx::mbar_wait(q_empty, (gu - 1) & 1);
      {
        const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(p.q) +
                                                          ((int64_t)token * p.hq + head) * D);
#pragma unroll
        for (int c = 0; c < D / 8; ++c) {
          uint4 v = r < u.n_rows ? __ldg(src + c) : make_uint4(0, 0, 0, 0);
          *reinterpret_cast<uint4*>(qs + (c / 8) * DN_CHUNK + ptx::sw128(r, c % 8)) = v;
        }
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(q_full);

      float m_ref = -INFINITY, l = 0.f;
      for (int j = 0; j < nb; ++j) {
        const uint32_t blk = gb + j, sb = blk & 1;
        // visible slots per entry of this block for this row
        int vis[EPB];
        bool full_vis = true;
#pragma unroll
        for (int i = 0; i < EPB; ++i) {
          const int e = u.entry_begin + j * EPB + i;
          int v = 0;
          if (e < u.entry_end) {
            const KvEntry en = p.entries[e];
            const int a = pos < en.pos0 ? 0 : pos - en.pos0 + 1;   // pos = INT32_MIN for padding rows
            v = a > en.count ? en.count : a;
          }
          vis[i] = v;
          full_vis = full_vis && (v == BOX);
        }
        ptx::mbar_wait(&s_full[sb], (blk >> 1) & 1);
        ptx::tc_fence_after();
        float s[DN_KB];
#pragma unroll
        for (int c = 0; c < DN_KB / 32; ++c)
          ptx::tmem_ld32(tmem + lane_base + sb * DN_KB + c * 32, reinterpret_cast<uint32_t*>(s + c * 32));
        ptx::tmem_wait_ld();
        float mx = -INFINITY;
        if (full_vis) {
#pragma unroll
          for (int k = 0; k < DN_KB; ++k) mx = fmaxf(mx, s[k]);
        } else {
#pragma unroll
          for (int k = 0; k < DN_KB; ++k) {
            s[k] = (k % BOX) < vis[k / BOX] ? s[k] : -INFINITY;
            mx = fmaxf(mx, s[k]);
          }
        }
        const float mx2 = mx * p.scale_log2;
        // PV of the previous block must be done before P smem / O are touched
        if (j > 0) ptx::mbar_wait(o_done, (blk - 1) & 1);
        const bool need = mx2 > m_ref + DN_RESCALE_T;
        if (j > 0 && __any_sync(0xffffffffu, need)) {
          ptx::tc_fence_after();
          const float alpha = need ? ptx::ex2(m_ref - mx2) : 1.f;
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            uint32_t ov[32];
            ptx::tmem_ld32(tmem + lane_base + 2 * DN_KB + c * 32, ov);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 32; ++k) ov[k] = __float_as_uint(__uint_as_float(ov[k]) * alpha);
            ptx::tmem_st32(tmem + lane_base + 2 * DN_KB + c * 32, ov);
          }
          ptx::tmem_wait_st();
        }
        if (need) {
          l *= ptx::ex2(m_ref - mx2);   // m_ref = -inf -> 0
          m_ref = mx2;
        }
        const float m_use = m_ref == -INFINITY ? 0.f : m_ref;
        float lsum = 0.f;
#pragma unroll
        for (int c = 0; c < DN_KB / 8; ++c) {
          float pv[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            pv[k] = ptx::ex2(fmaf(s[c * 8 + k], p.scale_log2, -m_use));
            lsum += pv[k];
          }
          uint4 w;
          w.x = ptx::pack_bf16(pv[0], pv[1]);
          w.y = ptx::pack_bf16(pv[2], pv[3]);
          w.z = ptx::pack_bf16(pv[4], pv[5]);
          w.w = ptx::pack_bf16(pv[6], pv[7]);
          *reinterpret_cast<uint4*>(ps_ + (c / 8) * DN_CHUNK + ptx::sw128(r, c % 8)) = w;
        }
        l += lsum;
        ptx::fence_proxy_async_smem();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(p_full);
      }
      // ---- epilogue
      const uint32_t last = gb + nb - 1;
      ptx::mbar_wait(o_done, last & 1);
      ptx::tc_fence_after();
      const float m_use = m_ref == -INFINITY ? 0.f : m_ref;
      const float inv = l > 0.f ? 1.f / l : 0.f;
      const float lse2 = l > 0.f ? m_use + log2f(l) : -INFINITY;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t ov[32];
        ptx::tmem_ld32(tmem + lane_base + 2 * DN_KB + c * 32, ov);
        ptx::tmem_wait_ld();
        if (tgt == PM_DIRECT) {
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.out) +
                                                ((int64_t)token * p.hq + head) * D + c * 32);
#pragma unroll
          for (int k = 0; k < 32; k += 8) {
            uint4 w;
            w.x = ptx::pack_bf16(__uint_as_float(ov[k]) * inv, __uint_as_float(ov[k + 1]) * inv);
            w.y = ptx::pack_bf16(__uint_as_float(ov[k + 2]) * inv, __uint_as_float(ov[k + 3]) * inv);
            w.z = ptx::pack_bf16(__uint_as_float(ov[k + 4]) * inv, __uint_as_float(ov[k + 5]) * inv);
            w.w = ptx::pack_bf16(__uint_as_float(ov[k + 6]) * inv, __uint_as_float(ov[k + 7]) * inv);
            dst[k / 8] = w;
          }
        } else if (tgt >= 0) {
          float4* dst = reinterpret_cast<float4*>(p.ws_o + ((int64_t)tgt * p.hq + head) * D + c * 32);
#pragma unroll
          for (int k = 0; k < 32; k += 4)
            dst[k / 4] = make_float4(__uint_as_float(ov[k]) * inv, __uint_as_float(ov[k + 1]) * inv,
                                     __uint_as_float(ov[k + 2]) * inv, __uint_as_float(ov[k + 3]) * inv);
        }
      }
      if (tgt == PM_DIRECT) p.lse[(int64_t)token * p.hq + head] = lse2 * kLn2;
      else if (tgt >= 0) p.ws_lse[(int64_t)tgt * p.hq + head] = lse2;
      ptx::tc_fence_before();
      gb += nb;
      ++gu;
    }
  }
  __syncwarp();       // lane 0 of the producer / MMA warps rejoins its warp before the CTA barrier
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, DN_TMEM_COLS);
  }
}

cudaError_t make_cache_tmap(CUtensorMap* m, const void* base, int64_t rows, int D, int box_rows);
int num_sms_cached();

template <int D, int BOX>
static cudaError_t launch_dense_db(const AttnParams& p, int64_t n_cache_pages, cudaStream_t st) {
  CUtensorMap tk, tv;
  const int64_t rows = n_cache_pages * p.hkv * p.ps;
  cudaError_t e = make_cache_tmap(&tk, p.k_cache, rows, D, BOX);
  if (e != cudaSuccess) return e;
  e = make_cache_tmap(&tv, p.v_cache, rows, D, BOX);
  if (e != cudaSuccess) return e;
  const size_t smem = dense_layout(D).total + 1024;
  e = cudaFuncSetAttribute(dense_kernel<D, BOX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int grid = p.n_units < num_sms_cached() ? p.n_units : num_sms_cached();
  dense_kernel<D, BOX><<<grid, DN_THREADS, smem, st>>>(tk, tv, p);
  return cudaPeekAtLastError();
}

template <int D>
static cudaError_t launch_dense_d(const AttnParams& p, int64_t n_cache_pages, cudaStream_t st) {
  if (p.ps >= 64) return launch_dense_db<D, 64>(p, n_cache_pages, st);
  if (p.ps == 32) return launch_dense_db<D, 32>(p, n_cache_pages, st);
  return launch_dense_db<D, 16>(p, n_cache_pages, st);
}

cudaError_t launch_generic(const AttnParams& p, cudaStream_t st);

cudaError_t launch_dense(const AttnParams& p, int64_t n_cache_pages, cudaStream_t st) {
  if (p.n_units <= 0) return cudaSuccess;
  if (p.kv_f32) return launch_generic(p, st);
  return p.d == 128 ? launch_dense_d<128>(p, n_cache_pages, st) : launch_dense_d<64>(p, n_cache_pages, st);
}

}  // namespace blend
