// umma_bench.cu — diagnostics (not part of the library): per-SM tcgen05.mma throughput of
// the instruction shapes the dense pass can use, to decide its block shape.
//   SS  M=128 N=64/128/256 K=16 (A and B from smem, 128B swizzle, K-major)
//   TS  M=128 N=64/128     K=16 (A from TMEM, B from smem; B K-major or MN-major)
// One CTA per SM, one elected thread issues ITER MMAs back to back into one TMEM
// accumulator and commits; clock64 around the issue..completion.  Values are zeros
// (throughput does not depend on them).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2411_16102_b200/csrc \
//        -I include scripts/umma_bench.cu -o /tmp/umma_bench && /tmp/umma_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace blend;

constexpr int ITER = 4096;

template <int N, bool TS, bool B_MN>
__global__ void __launch_bounds__(128, 1) bench(unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  ptx::fence_proxy_async_smem();
  if (warp == 0) ptx::tmem_alloc(&slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {
    const uint32_t leader = ptx::elect_one();
    const uint64_t ad = ptx::umma_desc_sw128(ptx::smem_u32(smem), 16, 1024);
    const uint64_t bd = B_MN ? ptx::umma_desc_sw128(ptx::smem_u32(smem + 32768), 8192, 1024)
                             : ptx::umma_desc_sw128(ptx::smem_u32(smem + 32768), 16, 1024);
    constexpr uint32_t idesc = ptx::umma_idesc_bf16(128, N, 0, B_MN ? 1 : 0);
    long long t0 = clock64();
    for (int i = 0; i < ITER; ++i) {
      const uint32_t k = i & 3;   // walk the K chunk like a real loop (32 B per K=16 step)
      if (TS)
        ptx::umma_ts_lohi(leader, tmem, tmem + 256 + k * 8, (uint32_t)bd + (k * (B_MN ? 16 * 128 : 32) >> 4),
                          (uint32_t)(bd >> 32), idesc, 1u);
      else
        ptx::umma_ss_lohi(leader, tmem, (uint32_t)ad + (k * 32 >> 4), (uint32_t)(ad >> 32),
                          (uint32_t)bd + (k * (B_MN ? 16 * 128 : 32) >> 4), (uint32_t)(bd >> 32), idesc, 1u);
    }
    ptx::umma_commit_if(leader, &bar);
    ptx::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

template <int N, bool TS, bool B_MN>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * sizeof(unsigned long long));
  auto k = bench<N, TS, B_MN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  for (int rep = 0; rep < 2; ++rep) k<<<148, 128, 80 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += (double)h[i];
  s /= 148;
  const double flop = 2.0 * 128 * N * 16 * ITER;
  printf("%-28s %s  cycles/MMA %6.2f  FLOP/clk/SM %7.1f\n", name, cudaGetErrorString(e), s / ITER, flop / s);
  cudaFree(d);
}

int main() {
  run<64, false, false>("SS 128x64x16  (QK, N=64)");
  run<128, false, false>("SS 128x128x16 (QK, N=128)");
  run<256, false, false>("SS 128x256x16");
  run<64, true, false>("TS 128x64x16  (A in TMEM)");
  run<128, true, false>("TS 128x128x16 (A in TMEM)");
  run<128, true, true>("TS 128x128x16 B MN (PV)");
  run<256, true, true>("TS 128x256x16 B MN");
  return 0;
}
