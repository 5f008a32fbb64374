// streamw.cu — streaming pass, warp-per-unit form (the default streaming kernel).
//
// Same contract as stream.cu (SMALL units: <= 16 rows of one kv head over their page
// entries; PAPER §2.3, §7.2), organised so that a unit never needs a
// CTA barrier: each of the 4 consumer warps owns whole units and a private 3-stage
// ring of 32-key K/V half-entries in shared memory; one TMA producer warp serves the
// four rings round-robin (non-blocking mbarrier.test_wait), loading only the 16-row
// groups that hold valid slots.  A warp keeps the unit's full online-softmax state
// (m, l, O[16 x D] in mma.sync fragments), so short decode units (~100-token private
// suffixes) cost no cross-warp merge and no named-barrier stalls, and long units
// (16K-token contexts) stream at HBM speed with 4 units in flight per SM.
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>

#include "blend.h"
#include "common.cuh"
#include "ptx.cuh"

namespace blend {

constexpr int SW_WARPS = 4;
constexpr int SW_THREADS = 32 * (SW_WARPS + 1);
constexpr int SW_STAGES = 3;
constexpr int SW_KEYS = 32;                  // keys per stage (half a 64-slot entry)
constexpr int SW_CHUNK = SW_KEYS * 128;      // 32 rows x 128 B

struct StreamWSmem {
  uint32_t ring0, ring_stride, stage_stride, q0, q_stride, bar, total;
};

__host__ __device__ inline StreamWSmem streamw_layout(int D) {
  StreamWSmem L;
  const uint32_t CH = D / 64;
  L.stage_stride = 2 * CH * SW_CHUNK;                  // K chunks then V chunks
  L.ring_stride = SW_STAGES * L.stage_stride;
  L.ring0 = 0;
  L.q0 = SW_WARPS * L.ring_stride;                     // per warp: 2 x CH x (16 rows x 128 B)
  L.q_stride = 2 * CH * 2048;
  L.bar = L.q0 + SW_WARPS * L.q_stride;
  L.total = L.bar + 2 * SW_WARPS * SW_STAGES * 8;
  return L;
}

template <int D>
__global__ void __launch_bounds__(SW_THREADS, 1)
    streamw_kernel(const __grid_constant__ CUtensorMap tmk32, const __grid_constant__ CUtensorMap tmv32,
                   const __grid_constant__ CUtensorMap tmk16, const __grid_constant__ CUtensorMap tmv16,
                   AttnParams p) {
  constexpr int CH = D / 64;
  constexpr int NT = D / 8;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const StreamWSmem L = streamw_layout(D);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar);     // [warp][stage]
  uint64_t* empty = full + SW_WARPS * SW_STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wstride = SW_WARPS * gridDim.x;
  ptx::pdl_launch_dependents();

  if (threadIdx.x == 0) {
    for (int i = 0; i < SW_WARPS * SW_STAGES; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();

  if (warp == SW_WARPS) {
    // ===================== TMA producer: 4 rings, round-robin =====================
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tmk32);
      ptx::tma_prefetch_desc(&tmv32);
      ptx::tma_prefetch_desc(&tmk16);
      ptx::tma_prefetch_desc(&tmv16);
      // Per-ring state lives in registers and the metadata of the next entry / next unit
      // is prefetched, so issuing a stage never waits on a dependent global load.
      int unit[SW_WARPS], e[SW_WARPS], eend[SW_WARPS], kvh[SW_WARPS], half[SW_WARPS];
      int4 cur[SW_WARPS], nxt[SW_WARPS], nu[SW_WARPS];   // KvEntry; next unit {eb, ee, kvh, -}
      uint32_t it[SW_WARPS];
      const int4* ents = reinterpret_cast<const int4*>(p.entries);
      auto load_unit = [&](int ui) -> int4 {
        if (ui >= p.n_units) return make_int4(0, 0, 0, -1);
        const Unit un = p.units[ui];
        return make_int4(un.entry_begin, un.entry_end, un.kvh, 0);
      };
      int active = 0;
#pragma unroll
      for (int w = 0; w < SW_WARPS; ++w) {
        unit[w] = blockIdx.x * SW_WARPS + w;
        it[w] = 0;
        half[w] = 0;
        const int4 u0 = load_unit(unit[w]);
        e[w] = u0.x;
        eend[w] = u0.y;
        kvh[w] = u0.z;
        if (unit[w] < p.n_units) {
          ++active;
          cur[w] = ents[e[w]];
          nxt[w] = e[w] + 1 < eend[w] ? ents[e[w] + 1] : make_int4(0, 0, 0, 0);
        }
        nu[w] = load_unit(unit[w] + wstride);
      }
      uint64_t idle_since = 0;
      while (active > 0) {
        bool progress = false;
#pragma unroll
        for (int w = 0; w < SW_WARPS; ++w) {
          if (unit[w] >= p.n_units) continue;
          const uint32_t s = it[w] % SW_STAGES, ph = (it[w] / SW_STAGES) & 1;
          if (!ptx::mbar_test_wait(&empty[w * SW_STAGES + s], ph ^ 1)) continue;
          progress = true;
          const int count = cur[w].w;
          const int left = count - half[w] * SW_KEYS;
          const int rows = ((left < SW_KEYS ? left : SW_KEYS) + 15) & ~15;
          const int32_t y = (cur[w].x * p.hkv + kvh[w]) * p.ps + cur[w].y + half[w] * SW_KEYS;
          uint8_t* st = smem + L.ring0 + w * L.ring_stride + s * L.stage_stride;
          uint64_t* fb = &full[w * SW_STAGES + s];
          ptx::mbar_arrive_expect_tx(fb, 2u * CH * rows * 128u);
#pragma unroll
          for (int c = 0; c < CH; ++c) {
            if (rows == SW_KEYS) {
              ptx::tma_load_2d(st + c * SW_CHUNK, &tmk32, fb, c * 64, y);
              ptx::tma_load_2d(st + (CH + c) * SW_CHUNK, &tmv32, fb, c * 64, y);
            } else {
              ptx::tma_load_2d(st + c * SW_CHUNK, &tmk16, fb, c * 64, y);
              ptx::tma_load_2d(st + (CH + c) * SW_CHUNK, &tmv16, fb, c * 64, y);
            }
          }
          ++it[w];
          if (++half[w] * SW_KEYS >= count) {
            half[w] = 0;
            if (++e[w] < eend[w]) {
              cur[w] = nxt[w];
              if (e[w] + 1 < eend[w]) nxt[w] = ents[e[w] + 1];
            } else {
              unit[w] += wstride;
              if (unit[w] < p.n_units) {
                e[w] = nu[w].x;
                eend[w] = nu[w].y;
                kvh[w] = nu[w].z;
                cur[w] = ents[e[w]];
                nxt[w] = e[w] + 1 < eend[w] ? ents[e[w] + 1] : make_int4(0, 0, 0, 0);
                nu[w] = load_unit(unit[w] + wstride);
              } else {
                --active;
              }
            }
          }
        }
        if (progress) {
          idle_since = 0;
        } else {   // watchdog: no ring has freed a stage for 10 s -> protocol bug, fail loudly
          const uint64_t now = ptx::globaltimer_ns();
          if (idle_since == 0) idle_since = now;
          else if (now - idle_since > 10000000000ull) __trap();
        }
      }
    }
    ptx::pdl_wait();   // this grid completes only after the (overlapped) dense grid has completed
    return;
  }

  // ===================== consumer warp: whole units =====================
  // The next unit's Q rows (cp.async into the other half of a double buffer) and row
  // metadata are fetched while the current unit streams, so a unit starts without a
  // dependent global-load round trip.
  const int g8 = lane >> 2, c4 = lane & 3;
  uint8_t* ring = smem + L.ring0 + warp * L.ring_stride;
  const uint32_t qs_u32 = ptx::smem_u32(smem + L.q0 + warp * L.q_stride);
  uint64_t* wfull = full + warp * SW_STAGES;
  uint64_t* wempty = empty + warp * SW_STAGES;
  uint32_t it = 0;
  constexpr int CPL = (16 * D / 8) / 32;   // 16-byte Q chunks per lane (row = lane / 2)

  struct RowMeta {
    RowInfo r0, r1;
    int32_t pos0, pos1;
  };
  auto fetch_q = [&](const Unit& un, int buf) {
    const int r = lane >> 1;
    const bool valid = r < un.n_rows;
    const __nv_bfloat16* src = reinterpret_cast<const __nv_bfloat16*>(p.q);
    if (valid) {
      const RowInfo ri = row_info(p, un, r);
      src += ((int64_t)ri.token * p.hq + ri.head) * D;
    }
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      const int unit16 = (lane & 1) * CPL + k;
      ptx::cp_async16_zfill(qs_u32 + buf * (CH * 2048) + (unit16 / 8) * 2048 + ptx::sw128(r, unit16 % 8),
                            src + 8 * unit16, valid);
    }
    ptx::cp_async_commit();
  };
  auto fetch_meta = [&](const Unit& un) {
    RowMeta m{{0, 0, 0}, {0, 0, 0}, INT32_MIN, INT32_MIN};
    if (g8 < un.n_rows) {
      m.r0 = row_info(p, un, g8);
      m.pos0 = p.tok_pos[m.r0.token];
    }
    if (g8 + 8 < un.n_rows) {
      m.r1 = row_info(p, un, g8 + 8);
      m.pos1 = p.tok_pos[m.r1.token];
    }
    return m;
  };

  int ui = blockIdx.x * SW_WARPS + warp;
  Unit u_next = ui < p.n_units ? p.units[ui] : Unit{};
  RowMeta meta_next{};
  if (ui < p.n_units) {
    fetch_q(u_next, 0);
    meta_next = fetch_meta(u_next);
  }
  for (int buf = 0; ui < p.n_units; ui += wstride, buf ^= 1) {
    const Unit u = u_next;
    const RowMeta meta = meta_next;
    ptx::cp_async_wait_group0();
    __syncwarp();
    uint32_t qa[D / 16][4];
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      const int mi = lane >> 3;
      const int row = (mi & 1) * 8 + (lane & 7);
      const int unit16 = 2 * kk + (mi >> 1);
      ptx::ldsm_x4(qs_u32 + buf * (CH * 2048) + (unit16 / 8) * 2048 + ptx::sw128(row, unit16 % 8), qa[kk][0],
                   qa[kk][1], qa[kk][2], qa[kk][3]);
    }
    __syncwarp();   // every lane's ldmatrix of this buffer is done before the next prefetch targets it later
    if (ui + wstride < p.n_units) {
      u_next = p.units[ui + wstride];
      fetch_q(u_next, buf ^ 1);
      meta_next = fetch_meta(u_next);
    }
    const RowInfo ri0 = meta.r0, ri1 = meta.r1;
    const int32_t pos0r = meta.pos0, pos1r = meta.pos1;

    float o[NT][4];
#pragma unroll
    for (int j = 0; j < NT; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

    for (int e = u.entry_begin; e < u.entry_end; ++e) {
      const KvEntry en = p.entries[e];
      for (int h = 0; h * SW_KEYS < en.count; ++h, ++it) {
        const uint32_t s = it % SW_STAGES, ph = (it / SW_STAGES) & 1;
        const int kbase = h * SW_KEYS;                 // slot of key 0 of this stage
        const int nvalid = en.count - kbase;           // >= 1
        ptx::mbar_wait(&wfull[s], ph);
        const uint32_t kst = ptx::smem_u32(ring + s * L.stage_stride);
        const uint32_t vst = kst + CH * SW_CHUNK;
        const int ntv = nvalid >= SW_KEYS ? 4 : (nvalid + 7) / 8;   // n-tiles holding valid keys
        const int nkv = nvalid > 16 ? 2 : 1;                         // 16-key k-steps for PV
        float sc[4][4];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          if (nt >= ntv) break;
#pragma unroll
          for (int kk = 0; kk < D / 16; kk += 2) {
            const int mi = lane >> 3;
            const int row = nt * 8 + (lane & 7);
            const int unit16 = 2 * kk + mi;
            uint32_t b0, b1, b2, b3;
            ptx::ldsm_x4(kst + (unit16 / 8) * SW_CHUNK + ptx::sw128(row, unit16 % 8), b0, b1, b2, b3);
            ptx::mma_bf16_16816(sc[nt], qa[kk], b0, b1);
            ptx::mma_bf16_16816(sc[nt], qa[kk + 1], b2, b3);
          }
        }
        float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int key = nt * 8 + 2 * c4 + c;          // key within the stage
            const int kp = en.pos0 + kbase + key;
            const bool kv = key < nvalid;
            sc[nt][c] = (kv && kp <= pos0r) ? sc[nt][c] * p.scale_log2 : -INFINITY;
            sc[nt][2 + c] = (kv && kp <= pos1r) ? sc[nt][2 + c] * p.scale_log2 : -INFINITY;
            mx0 = fmaxf(mx0, sc[nt][c]);
            mx1 = fmaxf(mx1, sc[nt][2 + c]);
          }
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
        const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
        const float mu0 = mn0 == -INFINITY ? 0.f : mn0, mu1 = mn1 == -INFINITY ? 0.f : mn1;
        const float al0 = ptx::ex2(m0 - mu0), al1 = ptx::ex2(m1 - mu1);
        m0 = mn0;
        m1 = mn1;
        float ps0 = 0.f, ps1 = 0.f;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            sc[nt][c] = ptx::ex2(sc[nt][c] - mu0);
            sc[nt][2 + c] = ptx::ex2(sc[nt][2 + c] - mu1);
            ps0 += sc[nt][c];
            ps1 += sc[nt][2 + c];
          }
        l0 = l0 * al0 + ps0;
        l1 = l1 * al1 + ps1;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          o[j][0] *= al0;
          o[j][1] *= al0;
          o[j][2] *= al1;
          o[j][3] *= al1;
        }
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          if (ks >= nkv) break;
          uint32_t pa[4];
          pa[0] = ptx::pack_bf16(sc[2 * ks][0], sc[2 * ks][1]);
          pa[1] = ptx::pack_bf16(sc[2 * ks][2], sc[2 * ks][3]);
          pa[2] = ptx::pack_bf16(sc[2 * ks + 1][0], sc[2 * ks + 1][1]);
          pa[3] = ptx::pack_bf16(sc[2 * ks + 1][2], sc[2 * ks + 1][3]);
#pragma unroll
          for (int j = 0; j < NT; j += 2) {
            const int mi = lane >> 3;
            const int row = ks * 16 + (mi & 1) * 8 + (lane & 7);
            const int unit16 = j + (mi >> 1);
            uint32_t b0, b1, b2, b3;
            ptx::ldsm_x4_t(vst + (unit16 / 8) * SW_CHUNK + ptx::sw128(row, unit16 % 8), b0, b1, b2, b3);
            ptx::mma_bf16_16816(o[j], pa, b0, b1);
            ptx::mma_bf16_16816(o[j + 1], pa, b2, b3);
          }
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&wempty[s]);
      }
    }
    // ---- unit end: rows g8 (o[.][0,1]) and g8+8 (o[.][2,3]) straight from the fragments
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
#pragma unroll
    for (int half_row = 0; half_row < 2; ++half_row) {
      const int r = g8 + 8 * half_row;
      if (r >= u.n_rows) continue;
      const RowInfo ri = half_row ? ri1 : ri0;
      const float l = half_row ? l1 : l0, m = half_row ? m1 : m0;
      const int32_t tgt = row_target(p, u, ri.tl);
      if (tgt == PM_SKIP) continue;
      const float inv = l > 0.f ? 1.f / l : 0.f;
      const float lse2 = l > 0.f ? (m == -INFINITY ? 0.f : m) + log2f(l) : -INFINITY;
      if (tgt == PM_DIRECT) {
        __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.out) + ((int64_t)ri.token * p.hq + ri.head) * D;
#pragma unroll
        for (int j = 0; j < NT; ++j)
          *reinterpret_cast<uint32_t*>(dst + 8 * j + 2 * c4) =
              ptx::pack_bf16(o[j][2 * half_row] * inv, o[j][2 * half_row + 1] * inv);
        if (c4 == 0) p.lse[(int64_t)ri.token * p.hq + ri.head] = lse2 * kLn2;
      } else {
        float* dst = p.ws_o + ((int64_t)tgt * p.hq + ri.head) * D;
#pragma unroll
        for (int j = 0; j < NT; ++j)
          *reinterpret_cast<float2*>(dst + 8 * j + 2 * c4) =
              make_float2(o[j][2 * half_row] * inv, o[j][2 * half_row + 1] * inv);
        if (c4 == 0) p.ws_lse[(int64_t)tgt * p.hq + ri.head] = lse2;
      }
    }
  }
  ptx::pdl_wait();
}

cudaError_t make_cache_tmap(CUtensorMap* m, const void* base, int64_t rows, int D, int box_rows);
cudaError_t set_smem_once(const void* func, size_t bytes);
int num_sms_cached();

template <int D>
static cudaError_t launch_streamw_d(const AttnParams& p, int64_t n_cache_pages, cudaStream_t st, bool overlap) {
  CUtensorMap tk32, tv32, tk16, tv16;
  const int64_t rows = n_cache_pages * p.hkv * p.ps;
  const int box = p.ps < SW_KEYS ? p.ps : SW_KEYS;   // ps = 16 -> 16-row boxes throughout
  cudaError_t e = make_cache_tmap(&tk32, p.k_cache, rows, D, box);
  if (e == cudaSuccess) e = make_cache_tmap(&tv32, p.v_cache, rows, D, box);
  if (e == cudaSuccess) e = make_cache_tmap(&tk16, p.k_cache, rows, D, 16);
  if (e == cudaSuccess) e = make_cache_tmap(&tv16, p.v_cache, rows, D, 16);
  if (e != cudaSuccess) return e;
  const size_t smem = streamw_layout(D).total + 1024;
  e = set_smem_once((const void*)streamw_kernel<D>, smem);
  if (e != cudaSuccess) return e;
  const int warps = (p.n_units + SW_WARPS - 1) / SW_WARPS;
  const int grid = warps < num_sms_cached() ? warps : num_sms_cached();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(SW_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = overlap ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, streamw_kernel<D>, tk32, tv32, tk16, tv16, p);
}

cudaError_t launch_streamw(const AttnParams& p, int64_t n_cache_pages, cudaStream_t st, bool overlap) {
  if (p.n_units <= 0) return cudaSuccess;
  return p.d == 128 ? launch_streamw_d<128>(p, n_cache_pages, st, overlap)
                    : launch_streamw_d<64>(p, n_cache_pages, st, overlap);
}

}  // namespace blend
