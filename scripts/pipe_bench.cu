// pipe_bench.cu — diagnostics (not part of the library): per-SM throughput of the
// instructions the dense softmax is made of (MUFU ex2, bf16x2 pack, FFMA2 / FADD2, the
// FMA-pipe exp2 polynomial) and the tcgen05.ld / st round trip, with W warps per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2411_16102_b200/csrc \
//        -I include scripts/pipe_bench.cu -o scripts/pipe_bench && scripts/pipe_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace blend;

constexpr int ITER = 2048;

template <int OP>
__global__ void __launch_bounds__(256, 1) bench(float* out, unsigned long long* cyc, float seed) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = seed * (threadIdx.x + i) * 1e-3f - 0.5f;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (OP == 0) a[i] = ptx::ex2(a[i]);                                   // MUFU.EX2
      if (OP == 1) acc ^= ptx::pack_bf16(a[i], a[(i + 1) & 15]), a[i] += 1e-7f;   // F2FP (+FADD)
      if (OP == 2) {                                                           // FFMA2
        uint64_t x = ptx::f2pack(a[i], a[(i + 1) & 15]);
        x = ptx::ffma2(x, x, x);
        ptx::f2unpack(x, a[i], a[(i + 1) & 15]);
      }
      if (OP == 3) {                                                           // exp2 polynomial (pair)
        uint64_t x = ptx::f2pack(a[i] * 1e-3f, a[(i + 1) & 15] * 1e-3f);
        x = ptx::exp2_poly2(x);
        float u, v;
        ptx::f2unpack(x, u, v);
        a[i] = u - v;
      }
      if (OP == 4) a[i] = a[i] * 1.0001f + 1e-7f;                              // scalar FFMA
    }
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + (float)acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int warps) {
  float* o;
  unsigned long long* c;
  cudaMalloc(&o, 148 * 1024 * sizeof(float));
  cudaMalloc(&c, 148 * sizeof(unsigned long long));
  for (int rep = 0; rep < 2; ++rep) bench<OP><<<148, warps * 32>>>(o, c, 1.f);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += (double)h[i];
  s /= 148;
  const double ops = (double)ITER * 16 * warps * 32;   // thread-ops per SM
  printf("%-26s warps/SM %2d %s  thread-ops/clk/SM %7.2f  (warp-instr cycles per SMSP %5.2f)\n", name, warps,
         cudaGetErrorString(e), ops / s, s / ((double)ITER * 16 * warps / 4));
  cudaFree(o);
  cudaFree(c);
}

int main() {
  for (int w : {4, 8}) {
    run<0>("MUFU.EX2", w);
    run<1>("F2FP pack bf16x2 (+FADD)", w);
    run<2>("FFMA2 (pairs)", w);
    run<3>("exp2 poly (pairs)", w);
    run<4>("FFMA", w);
  }
  return 0;
}
