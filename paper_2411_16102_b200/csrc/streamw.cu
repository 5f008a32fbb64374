// streamw.cu — streaming pass, warp-per-unit form (the default streaming kernel).
//
// Same contract as stream.cu (SMALL units: <= 16 rows of one kv head over their page
// entries; PAPER §2.3, §7.2), organised so that a unit never needs a
// CTA barrier: each of the 4 consumer warps owns whole units and a private 3-stage
// ring of 32-key K/V half-entries in shared memory, fed by its own TMA producer warp
// that loads only the 16-row groups holding valid slots.  A warp keeps the unit's full
// online-softmax state (m, l, O[16 x D] in mma.sync fragments), so short decode units
// (~100-token private suffixes) cost no cross-warp merge and no named-barrier stalls,
// and long units (16K-token contexts) stream at HBM speed with 4 units in flight per SM.
//
// Units are handed out dynamically (one global atomic counter, reset by the launch):
// the planner orders them longest-first, so this is greedy LPT, and CTAs that start
// late because the overlapped dense pass still occupies their SM simply take fewer
// units.  A ring's producer fetches unit k+1 while streaming unit k and announces it
// to its consumer through a two-slot smem queue, so the consumer prefetches the next
// unit's Q rows and row metadata while the current one streams.
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>

#include "blend.h"
#include "common.cuh"
#include "ptx.cuh"

namespace blend {

#ifndef BLEND_TRACE_STAGES
#define BLEND_TRACE_STAGES 0   // 1: per-stage stamps (stages 4..11 of ring 0) in the diagnostics trace
#endif

#ifndef SW_WARPS_CFG
#define SW_WARPS_CFG 4
#define SW_STAGES_CFG 3
#endif
#ifndef SW_EVICT_FIRST
#define SW_EVICT_FIRST 1   // streaming K/V loads carry an L2 evict-first policy
#endif
#ifndef SW_Q_AFTER
#define SW_Q_AFTER 1   // the next unit's Q rows are requested after this many stages of the current one
#endif
constexpr int SW_WARPS = SW_WARPS_CFG;                  // consumer warps = rings = producer warps
constexpr int SW_THREADS = 32 * (2 * SW_WARPS);
constexpr int SW_STAGES = SW_STAGES_CFG;
constexpr int SW_STATIC = 0;                 // statically assigned units per ring (0: all dynamic, measured best)
constexpr int SW_KEYS = 32;                  // keys per stage (half a 64-slot entry)
constexpr int SW_CHUNK = SW_KEYS * 128;      // 32 rows x 128 B

struct StreamWSmem {
  uint32_t ring0, ring_stride, stage_stride, q0, q_stride, bar, uq, total;
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
  L.uq = L.bar + 2 * SW_WARPS * SW_STAGES * 8 + 2 * SW_WARPS * 2 * 8;   // + unit-queue barriers
  L.total = L.uq + SW_WARPS * 2 * 16;
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
  uint64_t* uqf = empty + SW_WARPS * SW_STAGES;   // [ring][2] unit index announced
  uint64_t* uqe = uqf + SW_WARPS * 2;             // [ring][2] announcement consumed
  int4* uq = reinterpret_cast<int4*>(smem + L.uq);   // [ring][2] {unit (>= n_units: done), entry begin, count}
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) trace_stamp_s(p, 0);
  ptx::pdl_launch_dependents();

  if (threadIdx.x == 0) {
    for (int i = 0; i < SW_WARPS * SW_STAGES; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < SW_WARPS * 2; ++i) {
      ptx::mbar_init(&uqf[i], 1);
      ptx::mbar_init(&uqe[i], 1);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();

  if (warp >= SW_WARPS) {
    // ===================== TMA producer of ring w =====================
    const int w = warp - SW_WARPS;
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tmk32);
      ptx::tma_prefetch_desc(&tmv32);
      ptx::tma_prefetch_desc(&tmk16);
      ptx::tma_prefetch_desc(&tmv16);
      const int4* ents = reinterpret_cast<const int4*>(p.entries);
#if SW_EVICT_FIRST
      const uint64_t pol = ptx::l2_policy_evict_first();
#endif
      uint64_t* rfull = full + w * SW_STAGES;
      uint64_t* rempty = empty + w * SW_STAGES;
      uint8_t* ring = smem + L.ring0 + w * L.ring_stride;
      uint32_t a = 0, it = 0;
      // announcements carry {unit, first entry, entry count}: the consumer prefetches the
      // unit's rows and entries without a dependent global load
      auto announce = [&](int idx, const Unit& u) {
        const uint32_t s = a & 1, ph = (a >> 1) & 1;
        ptx::mbar_wait(&uqe[w * 2 + s], ph ^ 1);
        uq[w * 2 + s] = make_int4(idx, u.entry_begin, u.entry_end - u.entry_begin, 0);
        ptx::mbar_arrive(&uqf[w * 2 + s]);   // release: the consumer reads the slot after its wait
        ++a;
      };
      const int n = p.n_units;
      // Unit pipeline, two deep: while unit k's stages are issued, unit k+1 is known
      // (struct loaded, announced, first entry requested) and unit k+2's index is being
      // fetched from the counter, so no dependent global load sits between two units.
      // Units come from the counter (greedy LPT over the longest-first order); the first
      // SW_STATIC per ring may instead be assigned round-robin (0 measured best: rings on
      // SMs freed late by the overlapped dense grid should take fewer units).
      const int R = (int)gridDim.x * SW_WARPS, ring_id = (int)blockIdx.x * SW_WARPS + w;
      const int nstat = n / R < SW_STATIC ? n / R : SW_STATIC;
      int k_next = 0;   // units of this ring handed out so far
      auto fetch = [&]() -> int {
        const int k = k_next++;
        if (k < nstat) return k * R + ring_id;
        // plain atom (no warp aggregation: that would shuffle the result right away and
        // wait for it); the result is first used one unit later
        int v;
        asm volatile("atom.global.add.s32 %0, [%1], 1;" : "=r"(v) : "l"(p.sched) : "memory");
        return nstat * R + v;
      };
      int i_cur = fetch();
      int i_nxt = fetch();
      Unit u_cur = i_cur < n ? p.units[i_cur] : Unit{};
      announce(i_cur, u_cur);
      int4 cur = i_cur < n ? ents[u_cur.entry_begin] : make_int4(0, 0, 0, 0);
      while (i_cur < n) {
        Unit u_nxt{};
        int4 nfirst = make_int4(0, 0, 0, 0);
        int i_nn = n;
        if (i_nxt < n) u_nxt = p.units[i_nxt];   // requested now, used after the first stage's issue
        int phase = 1;   // 2: next unit announced, its first entry and the index after it requested
        auto advance = [&]() {
          if (phase == 1) {
            announce(i_nxt, u_nxt);
            if (i_nxt < n) {
              nfirst = ents[u_nxt.entry_begin];
              i_nn = fetch();
            }
            phase = 2;
          }
        };
        for (int e = u_cur.entry_begin; e < u_cur.entry_end; ++e) {
          const int4 nxt = e + 1 < u_cur.entry_end ? ents[e + 1] : make_int4(0, 0, 0, 0);
          const int count = cur.w;
          for (int h = 0; h * SW_KEYS < count; ++h, ++it) {
            const uint32_t s = it % SW_STAGES, ph = (it / SW_STAGES) & 1;
            ptx::mbar_wait(&rempty[s], ph ^ 1);
#if BLEND_TRACE_STAGES
            if (w == 0 && it >= 4 && it < 12) trace_stamp_s(p, 52 + (it - 4));
#endif
            const int left = count - h * SW_KEYS;
            const int rows = ((left < SW_KEYS ? left : SW_KEYS) + 15) & ~15;
            const int32_t y = (cur.x * p.hkv + u_cur.kvh) * p.ps + cur.y + h * SW_KEYS;
            uint8_t* st = ring + s * L.stage_stride;
            ptx::mbar_arrive_expect_tx(&rfull[s], 2u * CH * rows * 128u);
#pragma unroll
            for (int c = 0; c < CH; ++c) {
#if SW_EVICT_FIRST
              // a streaming unit's K/V (a request's private suffix) is read once: evict-first
              // (it need not displace the dense pass's re-read K/V from L2; measured: C2
              // streaming pass 35 -> 31 us, C4 neutral, C3 / C5 within 1 %)
              if (rows == SW_KEYS) {
                ptx::tma_load_2d_hint(st + c * SW_CHUNK, &tmk32, &rfull[s], c * 64, y, pol);
                ptx::tma_load_2d_hint(st + (CH + c) * SW_CHUNK, &tmv32, &rfull[s], c * 64, y, pol);
              } else {
                ptx::tma_load_2d_hint(st + c * SW_CHUNK, &tmk16, &rfull[s], c * 64, y, pol);
                ptx::tma_load_2d_hint(st + (CH + c) * SW_CHUNK, &tmv16, &rfull[s], c * 64, y, pol);
              }
#else
              if (rows == SW_KEYS) {
                ptx::tma_load_2d(st + c * SW_CHUNK, &tmk32, &rfull[s], c * 64, y);
                ptx::tma_load_2d(st + (CH + c) * SW_CHUNK, &tmv32, &rfull[s], c * 64, y);
              } else {
                ptx::tma_load_2d(st + c * SW_CHUNK, &tmk16, &rfull[s], c * 64, y);
                ptx::tma_load_2d(st + (CH + c) * SW_CHUNK, &tmv16, &rfull[s], c * 64, y);
              }
#endif
            }
            advance();   // one pipeline step per issued stage, after its loads are in flight
          }
          cur = nxt;
        }
        advance();
        i_cur = i_nxt;
        u_cur = u_nxt;
        cur = nfirst;
        i_nxt = i_nn;
      }
    }
    // Lanes 1..31 must not reach griddepcontrol.wait while lane 0 still issues loads:
    // the wait parks the whole warp until the dense grid completes (measured: the
    // producer stalled ~13 us on C2 and the overlap was lost).
    __syncwarp();
    ptx::pdl_wait();   // this grid completes only after the (overlapped) dense grid has completed
    return;
  }

  // ===================== consumer warp: whole units =====================
  // The next unit's Q rows (cp.async into the other half of a double buffer), row
  // descriptors and first 32 page entries (one per lane) are fetched while the current
  // unit streams, so a unit starts without a dependent global-load round trip.
  const int g8 = lane >> 2, c4 = lane & 3;
  uint8_t* ring = smem + L.ring0 + warp * L.ring_stride;
  const uint32_t qs_u32 = ptx::smem_u32(smem + L.q0 + warp * L.q_stride);
  uint64_t* wfull = full + warp * SW_STAGES;
  uint64_t* wempty = empty + warp * SW_STAGES;
  const int4* ents = reinterpret_cast<const int4*>(p.entries);
  uint32_t it = 0;
  constexpr int CPL = (16 * D / 8) / 32;   // 16-byte Q chunks per lane (row = lane / 2)

  uint32_t a = 0;
  auto next_index = [&]() -> int4 {   // the ring's next announced unit (x >= n_units: no more work)
    const uint32_t s = a & 1, ph = (a >> 1) & 1;
    ptx::mbar_wait(&uqf[warp * 2 + s], ph);
    const int4 ann = uq[warp * 2 + s];
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&uqe[warp * 2 + s]);
    ++a;
    return ann;
  };
  struct Pre {
    RowDesc d0, d1;        // rows g8 and g8 + 8 (softmax / output rows of this lane)
    int eb, ne;            // entry range
    int4 ebatch;           // entry eb + lane (lane < ne)
    int32_t qrow;          // q row of this lane's Q-copy row (lane / 2), -1: padding
  };
  // issue every metadata load of the announced unit (none is used here, so no stall)
  auto prefetch = [&](const int4 ann) -> Pre {
    Pre r;
    const RowDesc* rd = p.srows + (int64_t)ann.x * STREAM_ROWS;
    r.qrow = rd[lane >> 1].qrow;
    r.d0 = rd[g8];
    r.d1 = rd[g8 + 8];
    r.eb = ann.y;
    r.ne = ann.z;
    r.ebatch = lane < r.ne ? ents[r.eb + lane] : make_int4(0, 0, 0, 0);
    return r;
  };
  // the next unit's Q rows (cp.async into buffer buf), issued once the current unit's
  // first stage is done: by then its row descriptors have arrived
  auto issue_q = [&](const Pre& r, int buf) {
    const bool valid = r.qrow >= 0;
    const __nv_bfloat16* src = reinterpret_cast<const __nv_bfloat16*>(p.q) + (valid ? (int64_t)r.qrow * D : 0);
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      const int unit16 = (lane & 1) * CPL + k;
      ptx::cp_async16_zfill(qs_u32 + buf * (CH * 2048) + (unit16 / 8) * 2048 + ptx::sw128(lane >> 1, unit16 % 8),
                            src + 8 * unit16, valid);
    }
    ptx::cp_async_commit();
  };

  int4 nann = next_index();
  Pre pre{};
  if (nann.x < p.n_units) {
    pre = prefetch(nann);
    issue_q(pre, 0);
  }
  int tu = 0;   // diagnostics: units done by this warp
  for (int buf = 0; nann.x < p.n_units; buf ^= 1, ++tu) {
    if (warp == 0 && lane == 0) trace_stamp_s(p, 2 + 4 * tu);
    const Pre cu = pre;
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
    nann = next_index();
    bool q_pending = nann.x < p.n_units;
    int q_wait = 0;   // stages of this unit done (the next unit's Q is issued after SW_Q_AFTER)
    if (q_pending) pre = prefetch(nann);
    const int32_t pos0r = cu.d0.qrow >= 0 ? cu.d0.pos : INT32_MIN;
    const int32_t pos1r = cu.d1.qrow >= 0 ? cu.d1.pos : INT32_MIN;

    float o[NT][4];
#pragma unroll
    for (int j = 0; j < NT; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

    int4 eb_cur = cu.ebatch, eb_nxt = make_int4(0, 0, 0, 0);
    if (cu.ne > 32) eb_nxt = lane + 32 < cu.ne ? ents[cu.eb + 32 + lane] : make_int4(0, 0, 0, 0);
    for (int k = 0; k < cu.ne; ++k) {
      const int kl = k & 31;
      if (kl == 0 && k > 0) {   // next batch of 32 entries (prefetched one batch ahead)
        eb_cur = eb_nxt;
        if (k + 32 < cu.ne) eb_nxt = lane + k + 32 < cu.ne ? ents[cu.eb + k + 32 + lane] : make_int4(0, 0, 0, 0);
      }
      const int en_pos0 = __shfl_sync(0xffffffffu, eb_cur.z, kl);
      const int en_count = __shfl_sync(0xffffffffu, eb_cur.w, kl);
      for (int h = 0; h * SW_KEYS < en_count; ++h, ++it) {
        const uint32_t s = it % SW_STAGES, ph = (it / SW_STAGES) & 1;
        const int kbase = h * SW_KEYS;                 // slot of key 0 of this stage
        const int nvalid = en_count - kbase;           // >= 1
        ptx::mbar_wait(&wfull[s], ph);
        if (warp == 0 && lane == 0 && k == 0 && h == 0) trace_stamp_s(p, 3 + 4 * tu);
        // A partial stage loads whole 16-row groups: the V rows past the entry's count
        // (the tail of a node's last page) may hold anything, NaN included, and the PV
        // MMA multiplies them by P = 0 -> zero them (the K rows are masked by the select
        // below, which discards NaN scores).
        const bool tail = nvalid < SW_KEYS && (nvalid & 15) != 0;
        if (tail) {
          const int nz = 16 - (nvalid & 15);
          uint8_t* vz = ring + s * L.stage_stride + CH * SW_CHUNK + nvalid * 128;
          for (int u = lane; u < nz * CH * 8; u += 32) {
            const int row = u / (CH * 8), c = (u / 8) % CH, k16 = u % 8;
            *reinterpret_cast<uint4*>(vz + c * SW_CHUNK + row * 128 + k16 * 16) = make_uint4(0, 0, 0, 0);
          }
          __syncwarp();
        }
#if BLEND_TRACE_STAGES
        if (warp == 0 && lane == 0 && it >= 4 && it < 12) trace_stamp_s(p, 36 + (it - 4));
#endif
        const uint32_t kst = ptx::smem_u32(ring + s * L.stage_stride);
        const uint32_t vst = kst + CH * SW_CHUNK;
        const int ntv = nvalid >= SW_KEYS ? 4 : (nvalid + 7) / 8;   // n-tiles holding valid keys
        const int nkv = nvalid > 16 ? 2 : 1;                         // 16-key k-steps for PV
        float sc[4][4];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
        // k-steps outermost: the four n-tiles' MMA chains interleave (each sc[nt] still sums
        // its k-steps in ascending order), so consecutive MMAs are independent
        auto qk_step = [&](int nt, int kk) {
          const int mi = lane >> 3;
          const int row = nt * 8 + (lane & 7);
          const int unit16 = 2 * kk + mi;
          uint32_t b0, b1, b2, b3;
          ptx::ldsm_x4(kst + (unit16 / 8) * SW_CHUNK + ptx::sw128(row, unit16 % 8), b0, b1, b2, b3);
          ptx::mma_bf16_16816(sc[nt], qa[kk], b0, b1);
          ptx::mma_bf16_16816(sc[nt], qa[kk + 1], b2, b3);
        };
        if (ntv == 4) {
          // the four n-tiles' K fragments of a k-step pair are requested before any MMA uses
          // them (ldmatrix and mma.sync issue in source order)
#pragma unroll
          for (int kk = 0; kk < D / 16; kk += 2) {
            uint32_t kb[4][4];
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
              const int row = nt * 8 + (lane & 7);
              const int unit16 = 2 * kk + (lane >> 3);
              ptx::ldsm_x4(kst + (unit16 / 8) * SW_CHUNK + ptx::sw128(row, unit16 % 8), kb[nt][0], kb[nt][1], kb[nt][2],
                           kb[nt][3]);
            }
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) ptx::mma_bf16_16816(sc[nt], qa[kk], kb[nt][0], kb[nt][1]);
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) ptx::mma_bf16_16816(sc[nt], qa[kk + 1], kb[nt][2], kb[nt][3]);
          }
        } else {
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) {
            if (nt >= ntv) break;
#pragma unroll
            for (int kk = 0; kk < D / 16; kk += 2) qk_step(nt, kk);
          }
        }
        float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int key = nt * 8 + 2 * c4 + c;          // key within the stage
            const int kp = en_pos0 + kbase + key;
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
        if (p.stats != nullptr) {   // diagnostics: stages, and stages that rescale a live row's O
          const bool rs = (m0 != -INFINITY && mn0 > m0) || (m1 != -INFINITY && mn1 > m1);
          const bool any_rs = __any_sync(0xffffffffu, rs);
          if (lane == 0) {
            stat_add(p, STAT_STREAM_STAGES, 1);
            if (any_rs) stat_add(p, STAT_STREAM_RESCALE, 1);
            if (tail) stat_add(p, STAT_TAIL_ZEROED, 1);
          }
        }
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
          // V fragments of four 16-column pairs in flight before their MMAs
#pragma unroll
          for (int j0 = 0; j0 < NT; j0 += 8) {
            uint32_t vb[4][4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int mi = lane >> 3;
              const int row = ks * 16 + (mi & 1) * 8 + (lane & 7);
              const int unit16 = j0 + 2 * q + (mi >> 1);
              ptx::ldsm_x4_t(vst + (unit16 / 8) * SW_CHUNK + ptx::sw128(row, unit16 % 8), vb[q][0], vb[q][1], vb[q][2],
                             vb[q][3]);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              ptx::mma_bf16_16816(o[j0 + 2 * q], pa, vb[q][0], vb[q][1]);
              ptx::mma_bf16_16816(o[j0 + 2 * q + 1], pa, vb[q][2], vb[q][3]);
            }
          }
        }
        if (tail) ptx::fence_proxy_async_smem();   // generic zero stores before the next TMA write
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&wempty[s]);
#if BLEND_TRACE_STAGES
        if (warp == 0 && lane == 0 && it >= 4 && it < 12) trace_stamp_s(p, 44 + (it - 4));
#endif
        if (q_pending && ++q_wait >= SW_Q_AFTER) {
          issue_q(pre, buf ^ 1);
          q_pending = false;
        }
      }
    }
    if (q_pending) issue_q(pre, buf ^ 1);
    if (warp == 0 && lane == 0) trace_stamp_s(p, 4 + 4 * tu);
    // ---- unit end: rows g8 (o[.][0,1]) and g8+8 (o[.][2,3]) straight from the fragments
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
#pragma unroll
    for (int half_row = 0; half_row < 2; ++half_row) {
      const RowDesc d = half_row ? cu.d1 : cu.d0;
      if (d.qrow < 0 || d.target == PM_SKIP) continue;
      const float l = half_row ? l1 : l0, m = half_row ? m1 : m0;
      const float inv = l > 0.f ? 1.f / l : 0.f;
      const float lse2 = l > 0.f ? (m == -INFINITY ? 0.f : m) + log2f(l) : -INFINITY;
      if (d.target == PM_DIRECT) {
        __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.out) + (int64_t)d.qrow * D;
#pragma unroll
        for (int j = 0; j < NT; ++j)
          *reinterpret_cast<uint32_t*>(dst + 8 * j + 2 * c4) =
              ptx::pack_bf16(o[j][2 * half_row] * inv, o[j][2 * half_row + 1] * inv);
        if (c4 == 0) p.lse[d.qrow] = lse2 * kLn2;
      } else {
        float* dst = p.ws_o + ((int64_t)d.target * p.hq + d.head) * D;
#pragma unroll
        for (int j = 0; j < NT; ++j)
          *reinterpret_cast<float2*>(dst + 8 * j + 2 * c4) =
              make_float2(o[j][2 * half_row] * inv, o[j][2 * half_row + 1] * inv);
        if (c4 == 0) p.ws_lse[(int64_t)d.target * p.hq + d.head] = lse2;
      }
    }
    if (warp == 0 && lane == 0) trace_stamp_s(p, 5 + 4 * tu);
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
  int grid = warps < num_sms_cached() ? warps : num_sms_cached();
#ifdef SW_GRID_CAP
  if (grid > SW_GRID_CAP) grid = SW_GRID_CAP;   // diagnostics: bandwidth of the pass on fewer SMs
#endif
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
