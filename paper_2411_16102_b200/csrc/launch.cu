// launch.cu — host-side launch helpers shared by the kernels' launchers: TMA tensor-map
// encoding with a small cache (a steady-state blend_attention call only enqueues
// launches), per-(kernel, device) dynamic-smem attributes, and the SM count of the
// current device.  All caches are keyed by device (or by device pointer, which is
// unique per device under UVA) and guarded by one mutex, so a process may drive
// several GPUs from several threads.
#include <cuda.h>
#include <cuda_runtime.h>

#include <mutex>

#include "blend.h"
#include "common.cuh"

namespace blend {

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

namespace {
std::mutex g_mu;

PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;   // process-wide driver entry point (device independent)
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(ptr);
  }
  return fn;
}

struct TmapEntry {
  const void* base;
  int64_t rows;   // cache maps: rows; Q maps: tokens
  int kind;       // 0 cache map, 1 Q map
  int D, box, hq, g;
  CUtensorMap map;
};
constexpr int NTMAP = 48;
TmapEntry g_tmaps[NTMAP];
int g_tmap_n = 0, g_tmap_next = 0;

bool lookup(const TmapEntry& k, CUtensorMap* m) {
  for (int i = 0; i < g_tmap_n; ++i) {
    const TmapEntry& t = g_tmaps[i];
    if (t.base == k.base && t.rows == k.rows && t.kind == k.kind && t.D == k.D && t.box == k.box && t.hq == k.hq &&
        t.g == k.g) {
      *m = t.map;
      return true;
    }
  }
  return false;
}
void insert(const TmapEntry& k) {
  g_tmaps[g_tmap_next] = k;
  g_tmap_next = (g_tmap_next + 1) % NTMAP;
  if (g_tmap_n < NTMAP) ++g_tmap_n;
}

struct AttrEntry {
  const void* func;
  int device;
  size_t bytes;
};
AttrEntry g_attrs[64];
int g_attr_n = 0;
int g_sms[64];
}  // namespace

cudaError_t set_smem_once(const void* func, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mu);
  for (int i = 0; i < g_attr_n; ++i)
    if (g_attrs[i].func == func && g_attrs[i].device == dev && g_attrs[i].bytes >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess && g_attr_n < 64) g_attrs[g_attr_n++] = {func, dev, bytes};
  return e;
}

// 2-D view of a paged cache [pages*Hkv*ps rows][D] bf16, box {64 cols, box_rows}, 128B swizzle:
// one (page, kv head) block of a page is a run of ps rows, so a box is (part of) one page.
cudaError_t make_cache_tmap(CUtensorMap* m, const void* base, int64_t rows, int D, int box_rows) {
  std::lock_guard<std::mutex> lk(g_mu);
  TmapEntry k{base, rows, 0, D, box_rows, 0, 0, {}};
  if (lookup(k, m)) return cudaSuccess;
  PFN_encodeTiled enc = get_encode();
  if (!enc) return cudaErrorNotSupported;
  cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)D * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  k.map = *m;
  insert(k);
  return cudaSuccess;
}

// 3-D view of q [T][Hq][D] bf16, box {64 cols, g heads, box_tok tokens} (box_tok = 128/g:
// one 128-row dense Q tile chunk; 1: one token's g rows), 128B swizzle.
cudaError_t make_q_tmap(CUtensorMap* m, const void* base, int64_t T, int hq, int D, int g, int box_tok) {
  std::lock_guard<std::mutex> lk(g_mu);
  TmapEntry k{base, T, 1, D, box_tok, hq, g, {}};
  if (lookup(k, m)) return cudaSuccess;
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
  k.map = *m;
  insert(k);
  return cudaSuccess;
}

// SM count of the current device (cached per device).
int num_sms_cached() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_sms[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    g_sms[dev] = n > 0 ? n : 148;
  }
  return g_sms[dev];
}

}  // namespace blend
