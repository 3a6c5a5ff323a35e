// Microbenchmark: do SHFL.IDX and conflict-free LDS share one MIO throughput
// limit on sm_100a?  Each kernel: 32 warps/SM, a dependent-free mix per loop.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(1024) k(float* out, int iters) {
  __shared__ float s[1024];
  s[threadIdx.x] = threadIdx.x * 0.5f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  float reg = lane * 1.25f;
  unsigned idx = lane;
  for (int i = 0; i < iters; ++i) {
    idx = (idx * 5 + 3) & 31;  // conflict-free permutation each step
    if (MODE & 1) {
      a0 += s[(idx ^ 1) + 32 * (threadIdx.x >> 5)];
      a1 += s[(idx ^ 2) + 32 * (threadIdx.x >> 5)];
    }
    if (MODE & 2) {
      a2 += __shfl_sync(0xffffffffu, reg, idx ^ 4);
      a3 += __shfl_sync(0xffffffffu, reg, idx ^ 8);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 1024 * 4 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    float t[4] = {0, 0, 0, 0};
    auto run = [&](auto kern, int mi) {
      kern<<<148, 1024>>>(out, iters);
      cudaEventRecord(e0);
      kern<<<148, 1024>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&t[mi], e0, e1);
    };
    run(k<1>, 1);
    run(k<2>, 2);
    run(k<3>, 3);
    const double n = 148.0 * 32 * iters * 2;  // warp-instructions per kind
    printf("LDS only %.3f ms (%.2f warp-LDS/clk/SM @1.965GHz)\n", t[1], n / (t[1] * 1e-3) / 148 / 1.965e9);
    printf("SHFL only %.3f ms (%.2f warp-SHFL/clk/SM)\n", t[2], n / (t[2] * 1e-3) / 148 / 1.965e9);
    printf("LDS+SHFL %.3f ms (sum of singles %.3f, max %.3f)\n", t[3], t[1] + t[2], t[1] > t[2] ? t[1] : t[2]);
  }
  return 0;
}
