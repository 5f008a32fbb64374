// fill.cu — device implementation of the synthetic input generator
// (the numpy twin is synth/values.py — the two are checked
// bit-exactly against each other by tests/test_gpu_parity.py).  Bench/test
// infrastructure: fills the caller's K/V cache and Q, flushes L2.
#include <cuda_runtime.h>

#include "blend.h"
#include "common.cuh"

extern "C" int blend_internal_fail(int status, const char* msg);

namespace blend {

constexpr uint64_t KV_SALT = 0x5BD1E9955BD1E995ull;
constexpr uint64_t Q_SALT = 0xC2B2AE3D27D4EB4Full;

// grid: (n_pages, ps), block: Hkv*D threads (<= 1024) or looped
__global__ void fill_kv_kernel(void* kc, void* vc, int f32, int hkv, int kvh0, int D, int ps, const int32_t* page_ids,
                               const int32_t* page_count, const uint64_t* page_hash, uint64_t seed) {
  extern __shared__ uint64_t salt[];   // [2][hkv][D]
  const uint64_t seed_kv = seed ^ KV_SALT;
  const int n = 2 * hkv * D;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int kind = i / (hkv * D), rem = i % (hkv * D), kvh = rem / D, e = rem % D;
    salt[i] = mix64(seed_kv + ((uint64_t)((kind << 8) + kvh0 + kvh) << 12) + (uint64_t)e);
  }
  __syncthreads();
  const int64_t pi = blockIdx.x;
  const int s = blockIdx.y;
  const int64_t page = page_ids[pi];
  const bool valid = s < page_count[pi];
  const uint64_t h = valid ? page_hash[pi * ps + s] : 0;
  for (int i = threadIdx.x; i < hkv * D; i += blockDim.x) {
    int kvh = i / D, e = i % D;
    int64_t idx = ((page * hkv + kvh) * ps + s) * (int64_t)D + e;
    float kv = valid ? grid_val(mix64(h ^ salt[i])) : 0.f;
    float vv = valid ? grid_val(mix64(h ^ salt[hkv * D + i])) : 0.f;
    st_elem(kc, idx, kv, f32);
    st_elem(vc, idx, vv, f32);
  }
}

__global__ void fill_q_kernel(void* q, int f32, int hq, int h0, int D, const int64_t* row_gid, const int32_t* row_t,
                              uint64_t seed, float scale_q) {
  const int64_t row = blockIdx.x;
  const uint64_t seed_q = seed ^ Q_SALT;
  const uint64_t gid = (uint64_t)row_gid[row];
  const uint64_t t = (uint64_t)(uint32_t)row_t[row];
  for (int i = threadIdx.x; i < hq * D; i += blockDim.x) {
    uint64_t h = (uint64_t)(h0 + i / D), e = (uint64_t)(i % D);
    uint64_t ctr = ((gid * (1ull << 20) + t) * (1ull << 8) + h) * (1ull << 12) + e;
    float v = scale_q * grid_val(mix64(seed_q ^ mix64(ctr)));
    st_elem(q, row * (int64_t)hq * D + i, v, f32);
  }
}

__global__ void flush_kernel(uint4* p, size_t n, uint32_t salt) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(salt, (uint32_t)i, salt, 0);
}

}  // namespace blend

extern "C" int blend_fill_kv(void* k_cache, void* v_cache, int32_t kv_dtype, int32_t num_kv_heads, int32_t kv_head0,
                             int32_t head_dim, int32_t page_size, const int32_t* page_ids, const int32_t* page_count,
                             const uint64_t* page_hash, int64_t n_pages, uint64_t seed, void* stream) {
  if (!k_cache || !v_cache || !page_ids || !page_count || !page_hash)
    return blend_internal_fail(BLEND_EINVAL, "fill_kv: NULL argument");
  if (n_pages <= 0) return BLEND_OK;
  if (kv_head0 < 0 || kv_head0 + num_kv_heads > 256) return blend_internal_fail(BLEND_EINVAL, "fill_kv: kv heads");
  if (n_pages > 0x7fffffffLL || page_size > 65535) return blend_internal_fail(BLEND_EINVAL, "fill_kv: too many pages");
  dim3 grid((unsigned)n_pages, (unsigned)page_size);
  size_t smem = 2ull * num_kv_heads * head_dim * sizeof(uint64_t);
  if (smem > 48 * 1024) return blend_internal_fail(BLEND_EINVAL, "fill_kv: Hkv*D too large");
  blend::fill_kv_kernel<<<grid, 256, smem, (cudaStream_t)stream>>>(
      k_cache, v_cache, kv_dtype == BLEND_F32, num_kv_heads, kv_head0, head_dim, page_size, page_ids, page_count,
      page_hash, seed);
  if (cudaPeekAtLastError() != cudaSuccess) return blend_internal_fail(BLEND_ECUDA, cudaGetErrorString(cudaGetLastError()));
  return BLEND_OK;
}

extern "C" int blend_fill_q(void* q, int32_t dtype, int32_t num_q_heads, int32_t head0, int32_t head_dim,
                            const int64_t* row_gid, const int32_t* row_t, int64_t n_rows, uint64_t seed, float scale_q,
                            void* stream) {
  if (!q || !row_gid || !row_t) return blend_internal_fail(BLEND_EINVAL, "fill_q: NULL argument");
  if (n_rows <= 0) return BLEND_OK;
  if (head0 < 0 || head0 + num_q_heads > 256) return blend_internal_fail(BLEND_EINVAL, "fill_q: heads");
  if (n_rows > 0x7fffffffLL) return blend_internal_fail(BLEND_EINVAL, "fill_q: too many rows");
  blend::fill_q_kernel<<<(unsigned)n_rows, 256, 0, (cudaStream_t)stream>>>(q, dtype == BLEND_F32, num_q_heads,
                                                                           head0, head_dim, row_gid, row_t, seed,
                                                                           scale_q);
  if (cudaPeekAtLastError() != cudaSuccess) return blend_internal_fail(BLEND_ECUDA, cudaGetErrorString(cudaGetLastError()));
  return BLEND_OK;
}

extern "C" int blend_l2_flush(void* buf, size_t bytes, void* stream) {
  if (!buf) return blend_internal_fail(BLEND_EINVAL, "l2_flush: NULL buffer");
  static uint32_t salt = 1;
  blend::flush_kernel<<<148 * 4, 512, 0, (cudaStream_t)stream>>>((uint4*)buf, bytes / 16, salt++);
  if (cudaPeekAtLastError() != cudaSuccess) return blend_internal_fail(BLEND_ECUDA, cudaGetErrorString(cudaGetLastError()));
  return BLEND_OK;
}
