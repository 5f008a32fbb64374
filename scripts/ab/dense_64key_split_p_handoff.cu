// dense.cu — the dense pass on the 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// Work units with many rows per kv head — a SEPARATE shared-prefix node attended
// once by all the SMALL requests under it (PAPER §5 P:11 "exactly-once computation
// of shared prefixes"; §7.2 P:248-251 cascade reuse of the shared KV access), or a
// BIG request (chunked prefill) — are dense contractions: up to 256 query
// rows (tokens x grouped q heads) against 64-key blocks of the node's pages.
//
// One persistent CTA per SM, warp-specialised, two 128-row Q tiles (A, B) that
// share every K/V block ("ping-pong": the tensor pipe works on one tile while the
// other tile's softmax runs):
//   warp 0       TMA producer: 64-key K/V blocks (page entries, 128B swizzle) into a
//                4-stage smem ring
//   warp 1       MMA issuer (whole warp, one elected lane issues): S_t = Q_t K^T (UMMA
//                128x64x16, K-major A/B) into one of two TMEM S buffers per tile;
//                O_t += P_t V with P_t read from TMEM (aliasing its S buffer) and V
//                MN-major from smem; tcgen05.commit -> mbarriers
//   warp 2       TMEM allocator (512 columns: S_A0 S_A1 | S_B0 S_B1 | O_A | O_B)
//   warp 3       Q loader: the next unit's Q tiles as soon as the current unit's last
//                QK has been issued — 3-D TMA boxes {64, g, 128/g} when the unit's
//                tokens are consecutive rows of q, one box per token otherwise,
//                cp.async row gathers when g does not divide 128
//   warps 4..7   softmax / epilogue of tile A, warps 8..11 of tile B: thread =
//                query row = TMEM lane; tcgen05.ld the S row, per-row causal mask,
//                log2-domain online softmax with lazy O rescaling (only when the
//                running max grows by > 2^8; blocks whose exponentials sum to <= 2^8
//                against the running reference skip the block max), exp2 3/4 on
//                MUFU and 1/4 as an FMA-pipe polynomial, P -> bf16 -> tcgen05.st,
//                final O / l through a per-warp smem staging tile with coalesced
//                row-segment stores (bf16 output rows or fp32 partial rows).
// MMAs of one thread execute in issue order, so QK_t(j+2) (which overwrites the S
// buffer holding P_t(j)) is issued right after PV_t(j) without a further barrier.
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <string.h>

#include "blend.h"
#include "common.cuh"
#include "ptx.cuh"

namespace blend {

#ifndef DN_NSTAGE128
#define DN_NSTAGE128 4     // K/V ring stages at D = 128 (64 keys each)
#endif
#ifndef DN_REG_CTL
#define DN_REG_CTL 56      // setmaxnreg of warpgroup 0 (producer, MMA, allocator, Q loader)
#define DN_REG_SM 224      // setmaxnreg of the softmax warpgroups (56*128 + 224*256 = 64512)
#endif
#ifndef BLEND_TRACE_WARPS
#define BLEND_TRACE_WARPS 0    // 1: per-warp P hand-off stamps for blocks 20..23 of the first unit
#endif
#ifndef BLEND_TRACE_UNITS
#define BLEND_TRACE_UNITS 0    // 1: per-unit stamps (first 10 units of each CTA: start, first S, last P, epilogue end) and clock64 sums over all units
#endif
#ifndef BLEND_TRACE_BLOCKS
#define BLEND_TRACE_BLOCKS 0   // 1: per-block S / P stamps in the diagnostics trace (costs issue slots)
#endif

constexpr int DN_THREADS = 384;
constexpr int DN_KB = 64;                // keys per block (UMMA N of QK^T, K of PV)
constexpr int DN_QCHUNK = 128 * 128;     // Q: 128 rows x 128 B (one 64-column chunk)
constexpr int DN_KCHUNK = DN_KB * 128;   // K/V: 64 rows x 128 B
constexpr uint32_t DN_TMEM_COLS = 512;
constexpr float DN_RESCALE_T = 8.0f;     // lazy-rescale threshold (log2 units)

struct DenseSmem {
  uint32_t q0, q1, stage0, stage_stride, bar, stg, total;
  int nstage;
};

__host__ __device__ inline DenseSmem dense_layout(int D) {
  DenseSmem L;
  const int CH = D / 64;
  L.q0 = 0;
  L.q1 = CH * DN_QCHUNK;
  L.stage0 = 2 * CH * DN_QCHUNK;
  L.stage_stride = 2 * CH * DN_KCHUNK;   // K chunks then V chunks
  L.nstage = D == 128 ? DN_NSTAGE128 : 8;
  L.bar = L.stage0 + L.nstage * L.stage_stride;
  L.stg = L.bar + 512;                    // epilogue staging: per softmax warp 32 rows x 128 B
  L.total = L.stg + 8 * 4096;
  return L;
}

// The k-th unit of this CTA: units are sorted longest first and dealt out in a snake
// (round k even: CTA b takes k*G + b, odd: k*G + G-1-b), which balances the CTAs' totals
// far better than plain round robin (the longest of every round no longer lands on the
// same CTA).  Every warp of the CTA walks the same sequence.
__device__ __forceinline__ int snake_unit(int k) {
  const int G = (int)gridDim.x, b = (int)blockIdx.x;
  return k * G + ((k & 1) ? (G - 1 - b) : b);
}

// POLY: bit k set -> pair k (of 16 per 32-key chunk) takes the FMA-pipe polynomial exp2
#ifndef DN_POLY_MASK
#define DN_POLY_MASK 0x8888u   // pairs on the FMA-pipe polynomial: 4 of 16
#endif
template <int D, int BOX, uint32_t POLY = DN_POLY_MASK>
__global__ void __launch_bounds__(DN_THREADS, 1)
    dense_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                 const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmq1,
                 AttnParams p) {
  constexpr int CH = D / 64;
  constexpr int EPB = DN_KB / BOX;      // page entries per 64-key block
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const DenseSmem L = dense_layout(D);
  const int NS = L.nstage;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar);
  uint64_t* kv_full = bars;            // [NS <= 8]
  uint64_t* kv_empty = bars + 8;       // [NS]
  uint64_t* s_full = bars + 16;        // [tile][buffer]
  uint64_t* p_full = bars + 20;        // [tile][buffer]
  uint64_t* o_done = bars + 24;        // [tile][buffer]: PV of a block that used this S buffer
  uint64_t* q_full = bars + 28;
  uint64_t* q_empty = bars + 29;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 30);
  uint64_t* p_half = bars + 40;        // [tile][buffer]: P of the block's first 32 keys is in TMEM
  uint64_t* o_half = bars + 44;        // [tile][buffer]: PV of those 32 keys done

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) trace_stamp(p, 0);
  if (p.sched != nullptr && blockIdx.x == 0) {
    // reset the streaming pass's unit counter before this CTA's launch trigger: the
    // dependent (streaming) grid cannot start before every CTA of this grid has triggered
    if (threadIdx.x == 0) {
      if (atomicExch(p.sched, 0) == 0x7fffffff) __trap();   // consumes the result: the exchange has completed
      __threadfence();
    }
    __syncthreads();
  }
  ptx::pdl_launch_dependents();   // the streaming pass may start on SMs this grid leaves free
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      ptx::mbar_init(&kv_empty[s], 1);
    }
    for (int i = 0; i < 4; ++i) {
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&p_full[i], 4);
      ptx::mbar_init(&o_done[i], 1);
      ptx::mbar_init(&p_half[i], 4);
      ptx::mbar_init(&o_half[i], 1);
    }
    ptx::mbar_init(q_full, 1);
    ptx::mbar_init(q_empty, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, DN_TMEM_COLS);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) trace_stamp(p, 1);
  // TMEM columns: S[tile][buffer] 64 fp32 columns each at tile*128 + buffer*64 (P, bf16
  // pairs, aliases the first 32 columns of its S buffer); O[tile] at 256 + tile*D.
  // register budget: warpgroup 0 (producer, MMA, allocator, Q loader) needs few; the
  // softmax warpgroups get the rest of the CTA's launch allocation (168 x 384 = 64512 =
  // 56*128 + 224*256; setmaxnreg only redistributes the CTA's own registers).
  if (warp < 4) {
  ptx::setmaxnreg_dec<DN_REG_CTL>();
  if (warp == 0) {
    // ===================== TMA producer: 64-key K/V blocks into the stage ring =====================
    // The entries of the next block (and the next unit's header) are loaded one step
    // ahead, so a freed stage is refilled without waiting on dependent global loads.
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tmk);
      ptx::tma_prefetch_desc(&tmv);
      const int4* ents = reinterpret_cast<const int4*>(p.entries);
      uint32_t kit = 0;
      int uk = 0, ui = snake_unit(0);
      Unit u = ui < p.n_units ? p.units[ui] : Unit{};
      int4 cur[EPB];
      auto load_block = [&](const Unit& un, int j) {
#pragma unroll
        for (int i = 0; i < EPB; ++i) {
          int e = un.entry_begin + j * EPB + i;
          const bool pad = e >= un.entry_end;
          if (pad) e = un.entry_begin;                 // pad the last block (masked: count 0)
          cur[i] = ents[e];
          if (pad) cur[i].w = 0;
        }
      };
      if (ui < p.n_units) load_block(u, 0);
      while (ui < p.n_units) {
        const int nb = (u.entry_end - u.entry_begin + EPB - 1) / EPB;
        const int ui_next = snake_unit(++uk);
        const Unit un = ui_next < p.n_units ? p.units[ui_next] : Unit{};
        for (int j = 0; j < nb; ++j, ++kit) {
          const uint32_t s = kit % NS, ph = (kit / NS) & 1;
          ptx::mbar_wait(&kv_empty[s], ph ^ 1);
          uint8_t* kst = smem + L.stage0 + s * L.stage_stride;
          uint8_t* vst = kst + CH * DN_KCHUNK;
          if (kit == 0) trace_stamp(p, 3);
          ptx::mbar_arrive_expect_tx(&kv_full[s], 2u * CH * DN_KCHUNK);
#pragma unroll
          for (int i = 0; i < EPB; ++i) {
            const int32_t y = (cur[i].x * p.hkv + u.kvh) * p.ps + cur[i].y;   // {page, row_off, pos0, count}
#pragma unroll
            for (int c = 0; c < CH; ++c) {
              ptx::tma_load_2d(kst + c * DN_KCHUNK + i * BOX * 128, &tmk, &kv_full[s], c * 64, y);
              ptx::tma_load_2d(vst + c * DN_KCHUNK + i * BOX * 128, &tmv, &kv_full[s], c * 64, y);
            }
          }
          if (j + 1 < nb) load_block(u, j + 1);
          else if (ui_next < p.n_units) load_block(un, 0);
        }
        ui = ui_next;
        u = un;
      }
    }
  } else if (warp == 3) {
    // ===================== Q loader: next unit's rows as soon as its last QK is issued =====
    // A unit whose tokens are consecutive rows of q (a prefill chunk) loads each 128-row
    // tile chunk with one 3-D TMA box {64 cols, g heads, 128/g tokens}; other units (a
    // SEPARATE node's tokens come from many requests) gather rows with cp.async.
    if (lane == 0 && 128 % p.g == 0) {
      ptx::tma_prefetch_desc(&tmq);
      ptx::tma_prefetch_desc(&tmq1);
    }
    uint32_t gu = 0;
    for (int uk = 0, ui = snake_unit(0); ui < p.n_units; ui = snake_unit(++uk), ++gu) {
      const Unit u = p.units[ui];
      const int qt0 = p.dqtok[ui];
      if (gu > 0) ptx::mbar_wait(q_empty, (gu - 1) & 1);
      const int nrows = u.n_rows > 128 ? 256 : 128;
      if (qt0 >= 0) {
        if (lane == 0) {
          const int ntile = nrows >> 7;
          ptx::mbar_arrive_expect_tx(q_full, (uint32_t)(ntile * CH * DN_QCHUNK));
          for (int t = 0; t < ntile; ++t)
#pragma unroll
            for (int c = 0; c < CH; ++c)
              ptx::tma_load_3d(smem + (t ? L.q1 : L.q0) + c * DN_QCHUNK, &tmq, q_full, c * 64, u.kvh * p.g,
                               qt0 + t * (128 / p.g));
        }
        __syncwarp();
        continue;
      }
      if (128 % p.g == 0) {
        // tokens from many requests (a SEPARATE node): one TMA box {64, g, 1} per token and
        // 64-column chunk, issued by the lanes in parallel (each box = g whole rows)
        const int ntok = (u.n_rows + p.g - 1) / p.g, tpt = 128 / p.g;
        if (lane == 0) ptx::mbar_arrive_expect_tx(q_full, (uint32_t)(ntok * CH * p.g * 128));
        __syncwarp();
        for (int i = lane; i < ntok; i += 32) {
          const int tok = p.item_tokens[u.tok_base + u.row_begin / p.g + i];
          uint8_t* dst = smem + (i >= tpt ? L.q1 : L.q0) + (i % tpt) * p.g * 128;
#pragma unroll
          for (int c = 0; c < CH; ++c) ptx::tma_load_3d(dst + c * DN_QCHUNK, &tmq1, q_full, c * 64, u.kvh * p.g, tok);
        }
        continue;
      }
      // all of this lane's row tokens are requested before any is used (one round trip,
      // not one per row)
      int32_t qrow[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int row = lane + 32 * k;
        qrow[k] = -1;
        if (row < nrows && row < u.n_rows) {
          const int ir = u.row_begin + row, tl = ir / p.g;
          qrow[k] = p.item_tokens[u.tok_base + tl] * p.hq + u.kvh * p.g + (ir - tl * p.g);
        }
      }
#pragma unroll 1
      for (int k = 0; k < 8; ++k) {   // (the loader warp runs under setmaxnreg 56)
        const int row = lane + 32 * k;
        if (row >= nrows) break;
        uint8_t* qs = smem + ((row >> 7) ? L.q1 : L.q0);
        const int r = row & 127;
        if (qrow[k] >= 0) {
          const __nv_bfloat16* src = reinterpret_cast<const __nv_bfloat16*>(p.q) + (int64_t)qrow[k] * D;
#pragma unroll
          for (int c = 0; c < D / 8; ++c)
            ptx::cp_async16(qs + (c / 8) * DN_QCHUNK + ptx::sw128(r, c % 8), src + 8 * c);
        } else {
#pragma unroll
          for (int c = 0; c < D / 8; ++c)
            *reinterpret_cast<uint4*>(qs + (c / 8) * DN_QCHUNK + ptx::sw128(r, c % 8)) = make_uint4(0, 0, 0, 0);
        }
      }
      ptx::cp_async_wait_all();
      ptx::fence_proxy_async_smem();   // generic-proxy smem writes -> visible to the tensor core
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(q_full);
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (whole warp; one elected lane issues) =====================
    // Per unit: QK(0), QK(1) for every tile, then for j = 0..nb-1 and each tile:
    //   wait P_t(j) -> PV_t(j) (P from TMEM) -> commit o_done -> QK_t(j+2) into the S
    //   buffer PV_t(j) just consumed (MMAs execute in issue order) -> commit s_full.
    // The warp runs all lanes so descriptors stay warp-uniform; descriptors are built
    // once per stage and advanced by adding (byte offset >> 4) to the start-address field.
    {
      constexpr uint32_t IDESC_QK = ptx::umma_idesc_bf16(128, DN_KB, 0, 0);
      constexpr uint32_t IDESC_PV = ptx::umma_idesc_bf16(128, D, 0, 1);
      // descriptor halves: hi = SBO | version | swizzle (constant per operand kind),
      // lo = start address >> 4 | LBO >> 4 << 16, advanced by immediates
      const uint64_t qd0 = ptx::umma_desc_sw128(ptx::smem_u32(smem + L.q0), 16, 1024);
      const uint32_t q_lo0 = (uint32_t)qd0, q_hi = (uint32_t)(qd0 >> 32);
      const uint32_t q_lo1 = (uint32_t)ptx::umma_desc_sw128(ptx::smem_u32(smem + L.q1), 16, 1024);
      const uint64_t kd0 = ptx::umma_desc_sw128(ptx::smem_u32(smem + L.stage0), 16, 1024);
      const uint32_t k_lo0 = (uint32_t)kd0, k_hi = (uint32_t)(kd0 >> 32);
      const uint64_t vd0 = ptx::umma_desc_sw128(ptx::smem_u32(smem + L.stage0 + CH * DN_KCHUNK), DN_KCHUNK, 1024);
      const uint32_t v_lo0 = (uint32_t)vd0, v_hi = (uint32_t)(vd0 >> 32);
      const uint32_t stage_lo = L.stage_stride >> 4;
      const uint32_t leader = ptx::elect_one();
      uint32_t kit = 0, gu = 0;
      uint32_t pbits = 0;               // parity of the next p_full[tile][buffer] completion (bit pi)
      for (int uk = 0, ui = snake_unit(0); ui < p.n_units; ui = snake_unit(++uk)) {
        const Unit u = p.units[ui];
        const int nb = (u.entry_end - u.entry_begin + EPB - 1) / EPB;
        const int ntile = u.n_rows > 128 ? 2 : 1;
        auto wait_kv = [&](int j) {
          ptx::mbar_wait(&kv_full[(kit + j) % NS], ((kit + j) / NS) & 1);
          ptx::tc_fence_after();
        };
        auto issue_qk = [&](int t, int j) {
          const uint32_t qlo = t ? q_lo1 : q_lo0;
          const uint32_t klo = k_lo0 + ((kit + j) % NS) * stage_lo;
          const uint32_t dcol = tmem + t * 128 + (j & 1) * DN_KB;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            ptx::umma_ss_lohi(leader, dcol, qlo + (((kk / 4) * DN_QCHUNK + (kk % 4) * 32) >> 4), q_hi,
                              klo + (((kk / 4) * DN_KCHUNK + (kk % 4) * 32) >> 4), k_hi, IDESC_QK, kk > 0);
          ptx::umma_commit_if(leader, &s_full[t * 2 + (j & 1)]);
        };
        ptx::mbar_wait(q_full, gu & 1);
        ptx::tc_fence_after();
        if (gu == 0 && lane == 0) trace_stamp(p, 2);
        for (int j = 0; j < 2 && j < nb; ++j) {
          wait_kv(j);
          for (int t = 0; t < ntile; ++t) issue_qk(t, j);
        }
        if (nb <= 2) ptx::umma_commit_if(leader, q_empty);   // every QK of the unit issued: Q may be reloaded
        for (int j = 0; j < nb; ++j) {
          const uint32_t vlo = v_lo0 + ((kit + j) % NS) * stage_lo;
          if (j + 2 < nb) wait_kv(j + 2);
          for (int t = 0; t < ntile; ++t) {
            const int pi = t * 2 + (j & 1);
            const uint32_t acol = tmem + t * 128 + (j & 1) * DN_KB;
            // PV in two halves: the first 32 keys' P is handed over (p_half) while the softmax
            // still computes the second half, so the PV, and the QK behind it, start earlier
            ptx::mbar_wait(&p_half[pi], (pbits >> pi) & 1);
            ptx::tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < DN_KB / 32; ++kk)
              ptx::umma_ts_lohi(leader, tmem + 256 + t * D, acol + kk * 8, vlo + ((kk * 16 * 128) >> 4), v_hi,
                                IDESC_PV, (j > 0 || kk > 0) ? 1u : 0u);
            ptx::umma_commit_if(leader, &o_half[pi]);
            ptx::mbar_wait(&p_full[pi], (pbits >> pi) & 1);
            pbits ^= 1u << pi;
            ptx::tc_fence_after();
#pragma unroll
            for (int kk = DN_KB / 32; kk < DN_KB / 16; ++kk)
              ptx::umma_ts_lohi(leader, tmem + 256 + t * D, acol + kk * 8, vlo + ((kk * 16 * 128) >> 4), v_hi,
                                IDESC_PV, 1u);
            ptx::umma_commit_if(leader, &o_done[pi]);
            if (j + 2 < nb) issue_qk(t, j + 2);
          }
          if (j + 3 == nb) ptx::umma_commit_if(leader, q_empty);   // QK(nb-1) of every tile issued
          ptx::umma_commit_if(leader, &kv_empty[(kit + j) % NS]);
        }
        kit += nb;
        ++gu;
      }
    }
  }
  } else {
    ptx::setmaxnreg_inc<DN_REG_SM>();
    // ===================== softmax / epilogue (tile t) =====================
    const int t = (warp - 4) >> 2;                    // 0 = tile A, 1 = tile B
    const int r = threadIdx.x - 128 - 128 * t;        // row within the tile = TMEM lane
    const uint32_t lane_base = (uint32_t)(((warp - 4) & 3) * 32) << 16;
    const uint32_t col_o = 256 + t * D;
    uint32_t sb = 0;                                  // blocks of this tile processed so far
#if BLEND_TRACE_UNITS
    long long ph_acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};   // per fast block: two-tile [4], single-tile [4], counts [2]
    long long cu_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // clock64 sums: start->S0, S0->last P, epilogue, gap; blocks; units;
                                                      // single-tile units: S0->last P, blocks
    long long cu_prev_end = 0;
#endif
    uint32_t scnt0 = 0, scnt1 = 0;                    // s_full completions consumed per S buffer (registers)
    // {pos0, count} of the next block's entries, as loaded, and whether each is padding: the
    // padding select is applied when the block is processed, so no instruction waits on
    // the load right after issuing it
    int2 enext[EPB];
    bool epad[EPB];
    auto load_meta = [&](const Unit& un, int j) {
#pragma unroll
      for (int i = 0; i < EPB; ++i) {   // one 8-byte load per entry, no branch (padding: count 0)
        const int e = un.entry_begin + j * EPB + i;
        const int ec = e < un.entry_end ? e : un.entry_end - 1;
        enext[i] = *reinterpret_cast<const int2*>(&p.entries[ec].pos0);
        epad[i] = e >= un.entry_end;
      }
    };
    for (int uk = 0, ui = snake_unit(0); ui < p.n_units; ui = snake_unit(++uk)) {
      const Unit u = p.units[ui];
      const int nb = (u.entry_end - u.entry_begin + EPB - 1) / EPB;
      if (t == 1 && u.n_rows <= 128) continue;       // tile B idle for this unit
      const int row = 128 * t + r;                    // row within the unit
#if BLEND_TRACE_UNITS
      if (threadIdx.x == 128 && uk < 10) trace_stamp(p, 20 + 4 * uk);
      const long long cu0 = clock64();
      if (cu_prev_end != 0) cu_acc[3] += cu0 - cu_prev_end;
      long long cu_s0 = cu0;
#endif
      int32_t pos = INT32_MIN, token = 0, head = 0, tgt = PM_SKIP;
      if (row < u.n_rows) {
        // a TMA-loaded unit's tokens are consecutive from dqtok: no item_tokens round trip
        const int qt0 = p.dqtok[ui];
        const int ir = u.row_begin + row, tl = ir / p.g;
        tgt = row_target(p, u, tl);
        token = qt0 >= 0 ? qt0 + (tl - u.row_begin / p.g) : p.item_tokens[u.tok_base + tl];
        head = u.kvh * p.g + (ir - tl * p.g);
        pos = p.tok_pos[token];
      }
      float m_ref = -INFINITY, l = 0.f;
      const bool row_ok = row < u.n_rows;
      // a warp whose 32 rows are all padding (tile B of a 129..223-row unit) skips the
      // softmax: its P rows only feed its own (never stored) O rows, so they may hold
      // anything; it keeps the barrier protocol
      const bool warp_pad = __all_sync(0xffffffffu, !row_ok);
      load_meta(u, 0);
      for (int j = 0; j < nb; ++j, ++sb) {
        const int buf = j & 1;
        const uint32_t col_s = t * 128 + buf * DN_KB;
        // key positions of this block from the stage metadata the producer wrote (the
        // stage cannot be refilled before this block's P is consumed)
        // this block's {pos0, count} were loaded one block ahead (latency off the critical path)
        int2 ecur[EPB];
#pragma unroll
        for (int i = 0; i < EPB; ++i) ecur[i] = make_int2(enext[i].x, epad[i] ? 0 : enext[i].y);
        if (j + 1 < nb) load_meta(u, j + 1);
        int vis[EPB];
        bool full_vis = true;
#pragma unroll
        for (int i = 0; i < EPB; ++i) {
          const int2 en = ecur[i];                               // {pos0, count}
          const int a = pos < en.x ? 0 : pos - en.x + 1;          // pos = INT32_MIN for padding rows
          const int v = a > en.y ? en.y : a;
          vis[i] = v;
          full_vis = full_vis && (v == BOX);
        }
#if BLEND_TRACE_UNITS
        const long long ph0 = clock64();
#endif
        ptx::mbar_wait(&s_full[t * 2 + buf], (buf ? scnt1++ : scnt0++) & 1);   // per-buffer completion count
#if BLEND_TRACE_UNITS
        const long long ph1 = clock64();
#endif
        ptx::tc_fence_after();
#if BLEND_TRACE_UNITS
        if (threadIdx.x == 128 && uk < 10 && j == 0) trace_stamp(p, 21 + 4 * uk);
        if (j == 0) cu_s0 = clock64();
#endif
        // Entries with count < BOX (a node's last page, padding entries): their V rows past
        // the count may hold anything, NaN included, and the PV MMA would multiply them by
        // P = 0 -> tile A's warpgroup zeroes them before its P hand-off (the PV MMAs of both
        // tiles are issued after it).  K rows past the count only reach masked scores.
        if (t == 0) {
          bool part = false;
#pragma unroll
          for (int i = 0; i < EPB; ++i) part = part || ecur[i].y < BOX;
          if (part) {
            uint8_t* vst = smem + L.stage0 + (sb % NS) * L.stage_stride + CH * DN_KCHUNK;
#pragma unroll
            for (int i = 0; i < EPB; ++i) {
              const int nz = BOX - ecur[i].y;
              for (int x = r; x < nz * CH * 8; x += 128) {
                const int row = ecur[i].y + x / (CH * 8), c = (x / 8) % CH, k16 = x % 8;
                *reinterpret_cast<uint4*>(vst + c * DN_KCHUNK + (i * BOX + row) * 128 + k16 * 16) =
                    make_uint4(0, 0, 0, 0);
              }
            }
            ptx::fence_proxy_async_smem();   // generic stores -> visible to the tensor core (PV)
            if (r == 0) stat_add(p, STAT_TAIL_ZEROED, 1);
          }
        }
#if BLEND_TRACE_BLOCKS
        if (threadIdx.x == 128 && ui == (int)blockIdx.x) trace_stamp(p, 8 + 2 * j);
#endif
        if (warp_pad) {
          __syncwarp();
          if (lane == 0) {
            ptx::mbar_arrive(&p_half[t * 2 + buf]);
            ptx::mbar_arrive(&p_full[t * 2 + buf]);
          }
          continue;
        }
        float sv[DN_KB];
        ptx::tmem_ld32(tmem + lane_base + col_s, reinterpret_cast<uint32_t*>(sv));
        ptx::tmem_ld32(tmem + lane_base + col_s + 32, reinterpret_cast<uint32_t*>(sv + 32));
        ptx::tmem_wait_ld();
#if BLEND_TRACE_UNITS
        const long long ph2 = clock64();
        long long ph3 = ph2;
#endif
        if (!full_vis) {
#pragma unroll
          for (int k = 0; k < DN_KB; ++k) sv[k] = (k % BOX) < vis[k / BOX] ? sv[k] : -INFINITY;
        }
        // P = exp2(s*scale - m) on packed fp32 pairs (FFMA2/FADD2): 3 of every 4 pairs on the
        // MUFU pipe, 1 of 4 as a polynomial on the FMA pipe; bf16 pairs -> the first 32 TMEM
        // columns of this S buffer.
        uint32_t pk[DN_KB / 2];
        // one half of the block (16 pairs = 32 keys) against reference m_use; returns its sum
        auto exps_half = [&](float m_use, const int h) -> float {
          const uint64_t sc2 = ptx::f2pack(p.scale_log2, p.scale_log2), nm2 = ptx::f2pack(-m_use, -m_use);
          uint64_t ls2[2] = {ptx::f2pack(0.f, 0.f), ptx::f2pack(0.f, 0.f)};
#pragma unroll
          for (int k = 16 * h; k < 16 * h + 16; ++k) {
            const uint64_t x2 = ptx::ffma2(ptx::f2pack(sv[2 * k], sv[2 * k + 1]), sc2, nm2);
            uint64_t p2;
            if ((POLY >> (k & 15)) & 1u) {
              p2 = ptx::exp2_poly2(x2);
            } else {
              float x0, x1;
              ptx::f2unpack(x2, x0, x1);
              p2 = ptx::f2pack(ptx::ex2(x0), ptx::ex2(x1));
            }
            ls2[k & 1] = ptx::fadd2(ls2[k & 1], p2);
            float p0, p1;
            ptx::f2unpack(p2, p0, p1);
            pk[k] = ptx::pack_bf16(p0, p1);
          }
          float ls[4];
          ptx::f2unpack(ls2[0], ls[0], ls[1]);
          ptx::f2unpack(ls2[1], ls[2], ls[3]);
          return (ls[0] + ls[1]) + (ls[2] + ls[3]);
        };
        // hand over the P of half h: TMEM store, then the barrier the MMA warp waits on
        auto hand_half = [&](const int h, uint64_t* bar) {
          ptx::tmem_st16(tmem + lane_base + col_s + h * 16, pk + 16 * h);
          ptx::tmem_wait_st();
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(bar);
        };
        // rescale O (TMEM) by alpha once the PVs it holds are done (the caller waited)
        auto rescale_o = [&](float alpha) {
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            uint32_t ov[32];
            ptx::tmem_ld32(tmem + lane_base + col_o + c * 32, ov);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 32; ++k) ov[k] = __float_as_uint(__uint_as_float(ov[k]) * alpha);
            ptx::tmem_st32(tmem + lane_base + col_o + c * 32, ov);
          }
        };
        // Fast path: exponentiate against the running reference m_ref without the block
        // max.  Lazy rescaling keeps m_ref unless the max grows by more than 2^8, i.e. unless
        // some p > 2^8; a half's sum bounds each of its p, so lsum <= 2^8 proves that half
        // keeps m_ref and its P is exactly what the max-first order computes.  The first
        // half is handed to the MMA warp before the second is computed.  If the first half
        // fails (and on a unit's first block) the warp takes the max-first path below for
        // the whole block; if only the second fails, O (which then holds the first half's PV
        // against m_ref) is rescaled once that PV is done and the second half recomputed.
        const int pi = t * 2 + buf;
        bool slow = __any_sync(0xffffffffu, row_ok && m_ref == -INFINITY);
        bool late = false;
        if (!slow) {
          const float m_use = m_ref == -INFINITY ? 0.f : m_ref;   // -inf: a padding row (all scores masked)
          const float lsum0 = exps_half(m_use, 0);
          slow = __any_sync(0xffffffffu, !(lsum0 <= 256.f));
          if (!slow) {
            hand_half(0, &p_half[pi]);
            float lsum1 = exps_half(m_use, 1);
#if BLEND_TRACE_UNITS
            ph3 = clock64();
#endif
            late = __any_sync(0xffffffffu, !(lsum1 <= 256.f));
            l += lsum0;
            if (late) {
              float mxv[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) mxv[i] = sv[32 + i];
#pragma unroll
              for (int k = 36; k < DN_KB; ++k) mxv[k & 3] = fmaxf(mxv[k & 3], sv[k]);
              const float mx2 = fmaxf(fmaxf(mxv[0], mxv[1]), fmaxf(mxv[2], mxv[3])) * p.scale_log2;
              const bool need = mx2 > m_ref + DN_RESCALE_T;
              if (__any_sync(0xffffffffu, need)) {
                if (lane == 0) stat_add(p, STAT_DENSE_RESCALE, 1);
                // O holds every PV of the tile through this block's first half: wait for that
                // one (MMAs complete in issue order); its barrier completes once per use of
                // this S buffer, like s_full
                ptx::mbar_wait(&o_half[pi], ((buf ? scnt1 : scnt0) - 1) & 1);
                ptx::tc_fence_after();
                rescale_o(need ? ptx::ex2(m_ref - mx2) : 1.f);
              }
              if (need) {
                l *= ptx::ex2(m_ref - mx2);
                m_ref = mx2;
              }
              lsum1 = exps_half(m_ref == -INFINITY ? 0.f : m_ref, 1);
            }
            l += lsum1;
            hand_half(1, &p_full[pi]);
          }
        }
        if (p.stats != nullptr && lane == 0) {   // diagnostics: blocks per softmax path
          stat_add(p, STAT_DENSE_BLOCKS, 1);
          if (slow || late) stat_add(p, STAT_DENSE_SLOW, 1);
          if ((slow && j > 0) || late) stat_add(p, STAT_DENSE_SLOW_LATE, 1);
        }
        if (slow) {
        float mxv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) mxv[i] = sv[i];
#pragma unroll
        for (int k = 8; k < DN_KB; ++k) mxv[k & 7] = fmaxf(mxv[k & 7], sv[k]);
        const float mx = fmaxf(fmaxf(fmaxf(mxv[0], mxv[1]), fmaxf(mxv[2], mxv[3])),
                               fmaxf(fmaxf(mxv[4], mxv[5]), fmaxf(mxv[6], mxv[7])));
        const float mx2 = mx * p.scale_log2;
        const bool need = mx2 > m_ref + DN_RESCALE_T;
        if (j > 0 && __any_sync(0xffffffffu, need)) {
          if (lane == 0) stat_add(p, STAT_DENSE_RESCALE, 1);
          // O holds PV up to block j-1: wait for it.  Parity is unambiguous because the
          // previous completion on this barrier (PV(j-3)) is certified by s_full(j-1) and
          // PV(j+1) cannot be issued before this block's P.
          const int pb_ = (j - 1) & 1;
          ptx::mbar_wait(&o_done[t * 2 + pb_], ((pb_ ? scnt1 : scnt0) - 1) & 1);
          ptx::tc_fence_after();
          rescale_o(need ? ptx::ex2(m_ref - mx2) : 1.f);
        }
        if (need) {
          l *= ptx::ex2(m_ref - mx2);   // m_ref = -inf -> 0
          m_ref = mx2;
        }
          const float m_use = m_ref == -INFINITY ? 0.f : m_ref;
          l += exps_half(m_use, 0) + exps_half(m_use, 1);
          hand_half(0, &p_half[pi]);
          hand_half(1, &p_full[pi]);
        }
#if BLEND_TRACE_UNITS
        if (threadIdx.x == 128 && !slow) {
          const long long ph5 = clock64();
          const int k0 = u.n_rows <= 128 ? 52 : 48;   // [single-tile | two-tile]: s wait, ld, exps, st+arrive
          ph_acc[k0 - 48] += ph1 - ph0;
          ph_acc[k0 - 47] += ph2 - ph1;
          ph_acc[k0 - 46] += ph3 - ph2;
          ph_acc[k0 - 45] += ph5 - ph3;
          ph_acc[8 + (k0 == 52)] += 1;
        }
#endif
#if BLEND_TRACE_WARPS
        if (lane == 0 && ui == (int)blockIdx.x && j >= 20 && j < 24) trace_stamp(p, 24 + (j - 20) * 8 + (warp - 4));
#endif
#if BLEND_TRACE_BLOCKS
        if (threadIdx.x == 128 && ui == (int)blockIdx.x) trace_stamp(p, 9 + 2 * j);
#endif
      }
      if (threadIdx.x == 128 && ui == (int)blockIdx.x) trace_stamp(p, 4);
#if BLEND_TRACE_UNITS
      if (threadIdx.x == 128 && uk < 10) trace_stamp(p, 22 + 4 * uk);
      const long long cu_lp = clock64();
      cu_acc[0] += cu_s0 - cu0;
      cu_acc[1] += cu_lp - cu_s0;
      cu_acc[4] += nb;
      if (u.n_rows <= 128) {
        cu_acc[6] += cu_lp - cu_s0;
        cu_acc[7] += nb;
      }
      cu_acc[5] += 1;
#endif
      // ---- epilogue: PV of the unit's last block done (MMAs complete in issue order, so
      // this also certifies every earlier PV of the unit)
      {
        const int lb = (nb - 1) & 1;
        ptx::mbar_wait(&o_done[t * 2 + lb], ((lb ? scnt1 : scnt0) - 1) & 1);
      }
      ptx::tc_fence_after();
      if (threadIdx.x == 128 && ui == (int)blockIdx.x) trace_stamp(p, 60);
      const float m_use = m_ref == -INFINITY ? 0.f : m_ref;
      const float inv = l > 0.f ? 1.f / l : 0.f;
      const float lse2 = l > 0.f ? m_use + log2f(l) : -INFINITY;
      // O / l leaves through a per-warp smem staging tile (XOR-swizzled 16-B units, no
      // bank conflicts), so that every global store instruction writes whole row
      // segments of 4 rows instead of 32 scattered pieces.  Row kinds: 2 = fp32 partial
      // row, 1 = bf16 output row (DIRECT), 0 = nothing.  A warp whose rows are all bf16
      // outputs (or nothing) stages 64 columns as bf16 per pass (one 128-B line per row:
      // every STG.128 writes 4 whole lines); a warp with partial rows stages 32 fp32
      // columns per pass.
      {
        const int kind = tgt == PM_DIRECT ? 1 : (tgt >= 0 ? 2 : 0);
        char* rowp = kind == 1 ? reinterpret_cast<char*>(p.out) + ((int64_t)token * p.hq + head) * D * 2
                   : kind == 2 ? reinterpret_cast<char*>(p.ws_o + ((int64_t)tgt * p.hq + head) * D) : nullptr;
        const uint32_t stg = ptx::smem_u32(smem + L.stg + (warp - 4) * 4096);
        const int k8 = lane & 7;
        char* rp[8];
        int rk[8];
#pragma unroll
        for (int s_ = 0; s_ < 8; ++s_) {          // rows s_ * 4 + lane / 8 of this warp, for the copy-out
          const int rr = s_ * 4 + (lane >> 3);
          rp[s_] = reinterpret_cast<char*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(rowp), rr));
          rk[s_] = __shfl_sync(0xffffffffu, kind, rr);
        }
        const bool all_bf16 = __all_sync(0xffffffffu, kind != 2);
        // TMEM column loads two chunks at a time (one wait per 64 columns), then through
        // the staging tile
#pragma unroll 1
        for (int hh = 0; hh < D / 64; ++hh) {
         uint32_t ov2[64];
         ptx::tmem_ld32(tmem + lane_base + col_o + hh * 64, ov2);
         ptx::tmem_ld32(tmem + lane_base + col_o + hh * 64 + 32, ov2 + 32);
         ptx::tmem_wait_ld();
         if (hh == 0 && threadIdx.x == 128 && ui == (int)blockIdx.x) trace_stamp(p, 62);
         if (all_bf16) {
#pragma unroll
          for (int u8 = 0; u8 < 8; ++u8) {
            const uint32_t* o8 = ov2 + 8 * u8;
            ptx::sts128u(stg + ptx::sw128(lane, u8),
                         ptx::pack_bf16(__uint_as_float(o8[0]) * inv, __uint_as_float(o8[1]) * inv),
                         ptx::pack_bf16(__uint_as_float(o8[2]) * inv, __uint_as_float(o8[3]) * inv),
                         ptx::pack_bf16(__uint_as_float(o8[4]) * inv, __uint_as_float(o8[5]) * inv),
                         ptx::pack_bf16(__uint_as_float(o8[6]) * inv, __uint_as_float(o8[7]) * inv));
          }
          __syncwarp();
          uint4 v[8];   // all eight row segments in flight before the first store
#pragma unroll
          for (int s_ = 0; s_ < 8; ++s_) v[s_] = ptx::lds128u(stg + ptx::sw128(s_ * 4 + (lane >> 3), k8));
#pragma unroll
          for (int s_ = 0; s_ < 8; ++s_)
            if (rk[s_] == 1) ptx::stg128u(rp[s_] + hh * 128 + k8 * 16, v[s_]);
          __syncwarp();   // the staging tile is rewritten by the next chunk
          continue;
         }
#pragma unroll
         for (int cc = 0; cc < 2; ++cc) {
          const int c = 2 * hh + cc;
          const uint32_t* ov = ov2 + 32 * cc;
#pragma unroll
          for (int u8 = 0; u8 < 8; ++u8)
            ptx::sts128(stg + ptx::sw128(lane, u8), __uint_as_float(ov[4 * u8]) * inv,
                        __uint_as_float(ov[4 * u8 + 1]) * inv, __uint_as_float(ov[4 * u8 + 2]) * inv,
                        __uint_as_float(ov[4 * u8 + 3]) * inv);
          __syncwarp();
          float4 v[8];   // all eight row segments in flight before the first store
#pragma unroll
          for (int s_ = 0; s_ < 8; ++s_) v[s_] = ptx::lds128(stg + ptx::sw128(s_ * 4 + (lane >> 3), k8));
#pragma unroll
          for (int s_ = 0; s_ < 8; ++s_) {
            if (rk[s_] == 2)
              ptx::stg128(rp[s_] + c * 128 + k8 * 16, v[s_]);
            else if (rk[s_] == 1)
              ptx::stg64(rp[s_] + c * 64 + k8 * 8, ptx::pack_bf16(v[s_].x, v[s_].y), ptx::pack_bf16(v[s_].z, v[s_].w));
          }
          __syncwarp();   // the staging tile is rewritten by the next chunk
          if (c == 0 && threadIdx.x == 128 && ui == (int)blockIdx.x) trace_stamp(p, 63);
         }
        }
      }
      if (threadIdx.x == 128 && ui == (int)blockIdx.x) trace_stamp(p, 61);
      if (tgt == PM_DIRECT) p.lse[(int64_t)token * p.hq + head] = lse2 * kLn2;
      else if (tgt >= 0) p.ws_lse[(int64_t)tgt * p.hq + head] = lse2;
      ptx::tc_fence_before();
      if (threadIdx.x == 128 && ui == (int)blockIdx.x) trace_stamp(p, 5);
#if BLEND_TRACE_UNITS
      if (threadIdx.x == 128 && uk < 10) trace_stamp(p, 23 + 4 * uk);
      cu_prev_end = clock64();
      cu_acc[2] += cu_prev_end - cu_lp;
#endif
    }
#if BLEND_TRACE_UNITS
    if (threadIdx.x == 128 && p.trace != nullptr) {
      for (int i = 0; i < 8; ++i) p.trace[(size_t)blockIdx.x * 64 + 40 + i] = (unsigned long long)cu_acc[i];
      for (int i = 0; i < 10; ++i) p.trace[(size_t)blockIdx.x * 64 + 48 + i] = (unsigned long long)ph_acc[i];
    }
#endif
  }
  __syncwarp();       // lane 0 of the producer / MMA warps rejoins its warp before the CTA barrier
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) trace_stamp(p, 6);
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, DN_TMEM_COLS);
  }
}

cudaError_t make_cache_tmap(CUtensorMap* m, const void* base, int64_t rows, int D, int box_rows);
cudaError_t make_q_tmap(CUtensorMap* m, const void* base, int64_t T, int hq, int D, int g, int box_tok);
cudaError_t set_smem_once(const void* func, size_t bytes);
int num_sms_cached();

template <int D, int BOX>
static cudaError_t launch_dense_db(const AttnParams& p, int64_t n_cache_pages, cudaStream_t st) {
  CUtensorMap tk, tv;
  const int64_t rows = n_cache_pages * p.hkv * p.ps;
  cudaError_t e = make_cache_tmap(&tk, p.k_cache, rows, D, BOX);
  if (e != cudaSuccess) return e;
  e = make_cache_tmap(&tv, p.v_cache, rows, D, BOX);
  if (e != cudaSuccess) return e;
  CUtensorMap tq, tq1;   // Q boxes of 128/g tokens / of one token; only used when 128 % g == 0
  memset(&tq, 0, sizeof(tq));
  memset(&tq1, 0, sizeof(tq1));
  if (128 % p.g == 0) {
    e = make_q_tmap(&tq, p.q, p.n_tokens, p.hq, D, p.g, 128 / p.g);
    if (e == cudaSuccess) e = make_q_tmap(&tq1, p.q, p.n_tokens, p.hq, D, p.g, 1);
    if (e != cudaSuccess) return e;
  }
  const size_t smem = dense_layout(D).total + 1024;
  e = set_smem_once((const void*)dense_kernel<D, BOX>, smem);
  if (e != cudaSuccess) return e;
  int grid = p.n_units < num_sms_cached() ? p.n_units : num_sms_cached();
  if (p.dense_ctas > 0 && grid > p.dense_ctas) grid = p.dense_ctas;   // planner: SMs left to streaming
  dense_kernel<D, BOX><<<grid, DN_THREADS, smem, st>>>(tk, tv, tq, tq1, p);
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
