// stream.cu — the streaming pass: HBM-bound GQA attention of SMALL work units
// (<= 16 rows = query tokens x grouped q heads of one kv head) over their page
// entries, split-KV partials merged later by LSE.
//
// Per SURVEY §8(a-8) / PAPER §2.3 P:92-96 (decode "loads all p+i tokens"; with
// cascade the private part only, §7.2): the pass reads each K/V page-head
// block once per unit, so it is bound by HBM bandwidth.  Design (B200):
//   * persistent CTAs (1 per SM for long units, 2 per SM for short decode units),
//     static unit striding (units sorted longest first);
//   * a TMA producer warp streams 64-slot K/V page entries with
//     cp.async.bulk.tensor (128B swizzle) into an mbarrier ring of stages, loading
//     only the 16-row groups that hold valid slots of a partial page;
//   * 4 consumer warps split each stage's 64 keys (16 each): S = Q K^T and
//     O += P V on the legacy tensor pipe (mma.sync m16n8k16 bf16, fp32 accumulate;
//     at intensity g FLOP/B the FP32 FMA pipe would not keep up for g = 8),
//     warp-shuffle online softmax in the log2 domain;
//   * the 4 warp states are LSE-combined in shared memory at the unit end and
//     written as the final bf16 row (single-source token), an fp32 partial, or —
//     when the token's other sources are dense-pass partials — merged with those
//     in place (fused LSE merge, no separate merge launch for the token).
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>

#include <mutex>

#include "blend.h"
#include "common.cuh"
#include "ptx.cuh"

namespace blend {

constexpr int ST_CWARPS = 4;
constexpr int ST_THREADS = 32 * (ST_CWARPS + 1);
constexpr int ST_KEYS = 64;
constexpr int ST_CHUNK_BYTES = ST_KEYS * 128;   // one 64-col (128 B) chunk of 64 rows

struct StreamSmem {
  // byte offsets inside the dynamic smem block (base 1024-aligned)
  uint32_t stage0, stage_stride, q_off, merge_off, rowinfo_off, bar_off, total;
};

__host__ __device__ inline StreamSmem stream_smem_layout(int D, int nstage) {
  StreamSmem L;
  const uint32_t chunks = D / 64;
  L.stage0 = 0;
  L.stage_stride = 2 * chunks * ST_CHUNK_BYTES;               // K chunks then V chunks
  L.q_off = nstage * L.stage_stride;                          // Q: chunks x (16 rows x 128 B)
  L.merge_off = L.q_off + chunks * 2048;                      // 4 warps x (16 x D fp32 + 32 fp32)
  L.rowinfo_off = L.merge_off + ST_CWARPS * (16 * D + 32) * 4;
  L.bar_off = (L.rowinfo_off + 4 * 16 * 4 + 7) & ~7u;
  L.total = L.bar_off + 2 * nstage * 8;
  return L;
}

template <int D>
__global__ void __launch_bounds__(ST_THREADS, 2)
    stream_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                  const __grid_constant__ CUtensorMap tmk16, const __grid_constant__ CUtensorMap tmv16, AttnParams p,
                  int nstage, int box_rows) {
  constexpr int CH = D / 64;       // 128-B chunks per row
  constexpr int NT = D / 8;        // output n-tiles
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const StreamSmem L = stream_smem_layout(D, nstage);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* empty = full + nstage;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  ptx::pdl_launch_dependents();

  if (threadIdx.x == 0) {
    for (int s = 0; s < nstage; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], ST_CWARPS);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();

  if (warp == ST_CWARPS) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tmk);
      ptx::tma_prefetch_desc(&tmv);
      ptx::tma_prefetch_desc(&tmk16);
      ptx::tma_prefetch_desc(&tmv16);
      uint32_t it = 0;
      for (int ui = blockIdx.x; ui < p.n_units; ui += gridDim.x) {
        const Unit u = p.units[ui];
        for (int e = u.entry_begin; e < u.entry_end; ++e, ++it) {
          const uint32_t s = it % nstage, ph = (it / nstage) & 1;
          ptx::mbar_wait(&empty[s], ph ^ 1);
          const KvEntry en = p.entries[e];
          const int32_t y = (en.page * p.hkv + u.kvh) * p.ps + en.row_off;
          uint8_t* st = smem + L.stage0 + s * L.stage_stride;
          // load only the 16-row groups that hold valid slots (a node's last page is partial)
          const int rows = (en.count + 15) & ~15;
          ptx::mbar_arrive_expect_tx(&full[s], 2u * CH * rows * 128u);
          if (rows == box_rows) {
#pragma unroll
            for (int c = 0; c < CH; ++c) {
              ptx::tma_load_2d(st + c * ST_CHUNK_BYTES, &tmk, &full[s], c * 64, y);
              ptx::tma_load_2d(st + (CH + c) * ST_CHUNK_BYTES, &tmv, &full[s], c * 64, y);
            }
          } else {
            for (int r0 = 0; r0 < rows; r0 += 16)
#pragma unroll
              for (int c = 0; c < CH; ++c) {
                ptx::tma_load_2d(st + c * ST_CHUNK_BYTES + r0 * 128, &tmk16, &full[s], c * 64, y + r0);
                ptx::tma_load_2d(st + (CH + c) * ST_CHUNK_BYTES + r0 * 128, &tmv16, &full[s], c * 64, y + r0);
              }
          }
        }
      }
    }
    // Lanes 1..31 must not reach griddepcontrol.wait while lane 0 still issues loads:
    // the wait parks the whole warp until the dense grid completes (measured: the
    // producer stalled ~13 us on C2 and the overlap was lost).
    __syncwarp();
    ptx::pdl_wait();   // this grid completes only after the (overlapped) dense grid has completed
    return;
  }

  // ===================== consumers (4 warps) =====================
  const int tid = threadIdx.x;          // 0..127
  const int g8 = lane >> 2, c4 = lane & 3;
  uint8_t* qs = smem + L.q_off;
  float* mrg = reinterpret_cast<float*>(smem + L.merge_off);
  int32_t* rinfo = reinterpret_cast<int32_t*>(smem + L.rowinfo_off);   // [4][16]: pos, token, head, tgt
  const uint32_t qs_u32 = ptx::smem_u32(qs);
  uint32_t it = 0;

  for (int ui = blockIdx.x; ui < p.n_units; ui += gridDim.x) {
    const Unit u = p.units[ui];
    // ---- rows: metadata + Q tile (zero padded to 16 rows), 128B-swizzled
    if (tid < 16) {
      int32_t pos = INT32_MIN, token = 0, head = 0, tgt = PM_SKIP;
      if (tid < u.n_rows) {
        RowInfo ri = row_info(p, u, tid);
        pos = p.tok_pos[ri.token];
        token = ri.token;
        head = ri.head;
        tgt = row_target(p, u, ri.tl);
      }
      rinfo[tid] = pos;
      rinfo[16 + tid] = token;
      rinfo[32 + tid] = head;
      rinfo[48 + tid] = tgt;
    }
    for (int idx = tid; idx < 16 * (D / 8); idx += 128) {
      const int r = idx / (D / 8), unit = idx % (D / 8);
      uint4 v = make_uint4(0, 0, 0, 0);
      if (r < u.n_rows) {
        RowInfo ri = row_info(p, u, r);
        v = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(p.q) +
                                            ((int64_t)ri.token * p.hq + ri.head) * D + unit * 8);
      }
      *reinterpret_cast<uint4*>(qs + (unit / 8) * 2048 + ptx::sw128(r, unit % 8)) = v;
    }
    ptx::named_bar_sync(1, 128);
    uint32_t qa[D / 16][4];
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      const int mi = lane >> 3;
      const int row = (mi & 1) * 8 + (lane & 7);
      const int unit = 2 * kk + (mi >> 1);
      ptx::ldsm_x4(qs_u32 + (unit / 8) * 2048 + ptx::sw128(row, unit % 8), qa[kk][0], qa[kk][1], qa[kk][2],
                   qa[kk][3]);
    }
    const int32_t pos_g = rinfo[g8], pos_g8 = rinfo[g8 + 8];

    float o[NT][4];
#pragma unroll
    for (int j = 0; j < NT; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

    for (int e = u.entry_begin; e < u.entry_end; ++e, ++it) {
      const uint32_t s = it % nstage, ph = (it / nstage) & 1;
      const KvEntry en = p.entries[e];
      const int key0 = warp * 16;
      ptx::mbar_wait(&full[s], ph);
      if (key0 < box_rows && key0 < en.count) {
        const uint32_t kst = ptx::smem_u32(smem + L.stage0 + s * L.stage_stride);
        const uint32_t vst = kst + CH * ST_CHUNK_BYTES;
        float sc[2][4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < D / 16; kk += 2) {
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            const int mi = lane >> 3;
            const int row = key0 + nt * 8 + (lane & 7);
            const int unit = 2 * kk + mi;
            uint32_t b0, b1, b2, b3;
            ptx::ldsm_x4(kst + (unit / 8) * ST_CHUNK_BYTES + ptx::sw128(row, unit % 8), b0, b1, b2, b3);
            ptx::mma_bf16_16816(sc[nt], qa[kk], b0, b1);
            ptx::mma_bf16_16816(sc[nt], qa[kk + 1], b2, b3);
          }
        }
        // ---- mask + online softmax (log2 domain); rows g8 (regs 0,1) and g8+8 (regs 2,3)
        float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int key = key0 + nt * 8 + 2 * c4 + c;
            const int kp = en.pos0 + key;
            const bool kv = key < en.count;
            sc[nt][c] = (kv && kp <= pos_g) ? sc[nt][c] * p.scale_log2 : -INFINITY;
            sc[nt][2 + c] = (kv && kp <= pos_g8) ? sc[nt][2 + c] * p.scale_log2 : -INFINITY;
            mx0 = fmaxf(mx0, sc[nt][c]);
            mx1 = fmaxf(mx1, sc[nt][2 + c]);
          }
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
        const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
        const float mu0 = mn0 == -INFINITY ? 0.f : mn0, mu1 = mn1 == -INFINITY ? 0.f : mn1;
        const float al0 = exp2f(m0 - mu0), al1 = exp2f(m1 - mu1);
        m0 = mn0;
        m1 = mn1;
        float ps0 = 0.f, ps1 = 0.f;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            sc[nt][c] = exp2f(sc[nt][c] - mu0);
            sc[nt][2 + c] = exp2f(sc[nt][2 + c] - mu1);
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
        uint32_t pa[4];
        pa[0] = ptx::pack_bf16(sc[0][0], sc[0][1]);
        pa[1] = ptx::pack_bf16(sc[0][2], sc[0][3]);
        pa[2] = ptx::pack_bf16(sc[1][0], sc[1][1]);
        pa[3] = ptx::pack_bf16(sc[1][2], sc[1][3]);
        // ---- O += P V  (V via ldmatrix.trans)
#pragma unroll
        for (int j = 0; j < NT; j += 2) {
          const int mi = lane >> 3;
          const int row = key0 + (mi & 1) * 8 + (lane & 7);
          const int unit = j + (mi >> 1);
          uint32_t b0, b1, b2, b3;
          ptx::ldsm_x4_t(vst + (unit / 8) * ST_CHUNK_BYTES + ptx::sw128(row, unit % 8), b0, b1, b2, b3);
          ptx::mma_bf16_16816(o[j], pa, b0, b1);
          ptx::mma_bf16_16816(o[j + 1], pa, b2, b3);
        }
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&empty[s]);
    }

    // ---- unit end: combine the 4 warp states (LSE) and write the rows
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
    float* mw = mrg + warp * (16 * D + 32);
    if (c4 == 0) {
      mw[16 * D + g8] = m0;
      mw[16 * D + g8 + 8] = m1;
      mw[16 * D + 16 + g8] = l0;
      mw[16 * D + 16 + g8 + 8] = l1;
    }
    const bool w0 = g8 < u.n_rows, w1 = g8 + 8 < u.n_rows;   // padding rows are never read
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int d0 = 8 * j + 2 * c4;
      if (w0) *reinterpret_cast<float2*>(mw + g8 * D + d0) = make_float2(o[j][0], o[j][1]);
      if (w1) *reinterpret_cast<float2*>(mw + (g8 + 8) * D + d0) = make_float2(o[j][2], o[j][3]);
    }
    ptx::named_bar_sync(1, 128);
    {
      const int r = tid >> 3;                 // 16 rows x 8 threads
      const int dsl = (tid & 7) * (D / 8);    // D/8 elements per thread
      const int32_t tgt = rinfo[48 + r];
      if (r < u.n_rows && tgt != PM_SKIP) {
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < ST_CWARPS; ++w) M = fmaxf(M, mrg[w * (16 * D + 32) + 16 * D + r]);
        float coef[ST_CWARPS];
        float Lsum = 0.f;
#pragma unroll
        for (int w = 0; w < ST_CWARPS; ++w) {
          const float mwv = mrg[w * (16 * D + 32) + 16 * D + r];
          coef[w] = (M == -INFINITY) ? 0.f : exp2f(mwv - M);
          Lsum += coef[w] * mrg[w * (16 * D + 32) + 16 * D + 16 + r];
        }
        const float inv = Lsum > 0.f ? 1.f / Lsum : 0.f;
        const float lse2 = Lsum > 0.f ? M + log2f(Lsum) : -INFINITY;
        const int token = rinfo[16 + r], head = rinfo[32 + r];
        float ov[D / 8];
#pragma unroll
        for (int k = 0; k < D / 8; ++k) {
          float a = 0.f;
#pragma unroll
          for (int w = 0; w < ST_CWARPS; ++w) a += coef[w] * mrg[w * (16 * D + 32) + r * D + dsl + k];
          ov[k] = a * inv;
        }
        if (tgt <= PM_FUSED_BASE) {
          fused_merge_store(p, tgt, token, head, ov, lse2, dsl, 1, D / 8, (tid & 7) == 0);
        } else if (tgt == PM_DIRECT) {
          __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.out) + ((int64_t)token * p.hq + head) * D + dsl;
#pragma unroll
          for (int k = 0; k < D / 8; k += 8) {
            uint4 v;
            v.x = ptx::pack_bf16(ov[k], ov[k + 1]);
            v.y = ptx::pack_bf16(ov[k + 2], ov[k + 3]);
            v.z = ptx::pack_bf16(ov[k + 4], ov[k + 5]);
            v.w = ptx::pack_bf16(ov[k + 6], ov[k + 7]);
            *reinterpret_cast<uint4*>(dst + k) = v;
          }
          if ((tid & 7) == 0) p.lse[(int64_t)token * p.hq + head] = lse2 * kLn2;
        } else {
          float* dst = p.ws_o + ((int64_t)tgt * p.hq + head) * D + dsl;
#pragma unroll
          for (int k = 0; k < D / 8; k += 4) *reinterpret_cast<float4*>(dst + k) = make_float4(ov[k], ov[k + 1], ov[k + 2], ov[k + 3]);
          if ((tid & 7) == 0) p.ws_lse[(int64_t)tgt * p.hq + head] = lse2;
        }
      }
    }
    ptx::named_bar_sync(1, 128);
  }
  ptx::pdl_wait();
}

// ------------------------------------------------------------------ host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(ptr);
  }
  return fn;
}

// Host-side caches: tensor maps keyed by (base, rows, D, box) and per-kernel smem
// attributes, so a steady-state blend_attention call only enqueues launches.
namespace {
struct TmapEntry {
  const void* base;
  int64_t rows;
  int D, box;
  CUtensorMap map;
};
std::mutex g_cache_mu;
TmapEntry g_tmaps[32];
int g_tmap_n = 0, g_tmap_next = 0;
struct AttrEntry {
  const void* func;
  int device;
  size_t bytes;
};
AttrEntry g_attrs[32];
int g_attr_n = 0;
}  // namespace

cudaError_t set_smem_once(const void* func, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  for (int i = 0; i < g_attr_n; ++i)
    if (g_attrs[i].func == func && g_attrs[i].device == dev && g_attrs[i].bytes >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess && g_attr_n < 32) g_attrs[g_attr_n++] = {func, dev, bytes};
  return e;
}

static cudaError_t encode_cache_tmap(CUtensorMap* m, const void* base, int64_t rows, int D, int box_rows);

// 2-D view of a paged cache [pages*Hkv*ps rows][D] bf16, box {64 cols, box_rows}, 128B swizzle
cudaError_t make_cache_tmap(CUtensorMap* m, const void* base, int64_t rows, int D, int box_rows) {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  for (int i = 0; i < g_tmap_n; ++i) {
    const TmapEntry& t = g_tmaps[i];
    if (t.base == base && t.rows == rows && t.D == D && t.box == box_rows) {
      *m = t.map;
      return cudaSuccess;
    }
  }
  cudaError_t e = encode_cache_tmap(m, base, rows, D, box_rows);
  if (e != cudaSuccess) return e;
  TmapEntry& t = g_tmaps[g_tmap_next];
  t = {base, rows, D, box_rows, *m};
  g_tmap_next = (g_tmap_next + 1) % 32;
  if (g_tmap_n < 32) ++g_tmap_n;
  return cudaSuccess;
}

static cudaError_t encode_cache_tmap(CUtensorMap* m, const void* base, int64_t rows, int D, int box_rows) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return cudaErrorNotSupported;
  cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)D * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// 3-D view of q [T][Hq][D] bf16, box {64 cols, g heads, 128/g tokens} (one 128-row
// dense Q tile chunk), 128B swizzle.  Cached like the cache maps.
namespace {
struct QmapEntry {
  const void* base;
  int64_t T;
  int hq, D, g, bt;
  CUtensorMap map;
};
QmapEntry g_qmaps[8];
int g_qmap_n = 0, g_qmap_next = 0;
}  // namespace

cudaError_t make_q_tmap(CUtensorMap* m, const void* base, int64_t T, int hq, int D, int g, int box_tok) {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  for (int i = 0; i < g_qmap_n; ++i) {
    const QmapEntry& t = g_qmaps[i];
    if (t.base == base && t.T == T && t.hq == hq && t.D == D && t.g == g && t.bt == box_tok) {
      *m = t.map;
      return cudaSuccess;
    }
  }
  PFN_encodeTiled enc = get_encode();
  if (!enc) return cudaErrorNotSupported;
  cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)hq, (cuuint64_t)(T > 0 ? T : 1)};
  cuuint64_t strides[2] = {(cuuint64_t)D * 2, (cuuint64_t)hq * D * 2};
  cuuint32_t box[3] = {64, (cuuint32_t)g, (cuuint32_t)box_tok};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  QmapEntry& t = g_qmaps[g_qmap_next];
  t = {base, T, hq, D, g, box_tok, *m};
  g_qmap_next = (g_qmap_next + 1) % 8;
  if (g_qmap_n < 8) ++g_qmap_n;
  return cudaSuccess;
}

int num_sms_cached() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int D>
static cudaError_t launch_stream_d(const AttnParams& p, int64_t n_cache_pages, cudaStream_t st, bool overlap) {
  const int box_rows = p.ps < ST_KEYS ? p.ps : ST_KEYS;
  CUtensorMap tk, tv, tk16, tv16;
  const int64_t rows = n_cache_pages * p.hkv * p.ps;
  cudaError_t e = make_cache_tmap(&tk, p.k_cache, rows, D, box_rows);
  if (e == cudaSuccess) e = make_cache_tmap(&tv, p.v_cache, rows, D, box_rows);
  if (e == cudaSuccess) e = make_cache_tmap(&tk16, p.k_cache, rows, D, 16);
  if (e == cudaSuccess) e = make_cache_tmap(&tv16, p.v_cache, rows, D, 16);
  if (e != cudaSuccess) return e;
  // Short units (decode over a ~100-token private suffix): 2 CTAs per SM with a 2-stage
  // ring each, so one CTA's per-unit prologue/epilogue overlaps the other's streaming.
  // Long units (16K-token contexts): 1 CTA per SM with the deepest ring that fits.
  const int64_t avg_entries = p.avg_entries;
  int ctas_per_sm = avg_entries <= 8 ? 2 : 1;
  int nstage = ctas_per_sm == 2 ? 2 : 6;
  const int budget = ctas_per_sm == 2 ? 113 * 1024 : 227 * 1024;
  while (nstage > 2 && (int)stream_smem_layout(D, nstage).total + 1024 > budget) --nstage;
  const size_t smem = stream_smem_layout(D, nstage).total + 1024;
  e = set_smem_once((const void*)stream_kernel<D>, smem);
  if (e != cudaSuccess) return e;
  const int slots = ctas_per_sm * num_sms_cached();
  const int grid = p.n_units < slots ? p.n_units : slots;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(ST_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = overlap ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, stream_kernel<D>, tk, tv, tk16, tv16, p, nstage, box_rows);
}

cudaError_t launch_generic(const AttnParams& p, cudaStream_t st);

cudaError_t launch_stream(const AttnParams& p, int64_t n_cache_pages, cudaStream_t st, bool overlap) {
  if (p.n_units <= 0) return cudaSuccess;
  if (p.kv_f32) return launch_generic(p, st);
  return p.d == 128 ? launch_stream_d<128>(p, n_cache_pages, st, overlap)
                    : launch_stream_d<64>(p, n_cache_pages, st, overlap);
}

}  // namespace blend
