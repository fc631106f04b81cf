// Microbenchmark: does SHFL share the shared-memory data pipe with LDS?
// Kernel L: 4 independent LDS.32 chains per iteration; S: 4 SHFL chains;
// LS: both.  If LS time ~ max(L, S) the pipes are separate; ~ L + S shared.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void __launch_bounds__(512) kern(int iters, int* out) {
  __shared__ int sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i * 7;
  __syncthreads();
  int a = threadIdx.x, b = threadIdx.x + 1, c = threadIdx.x + 2, d = threadIdx.x + 3;
  int e = threadIdx.x, f = 5, g2 = 6, h = 7;
  for (int i = 0; i < iters; ++i) {
    if (MODE & 1) {
      a = sm[(a & 31) + (threadIdx.x & ~31)];
      b = sm[(b & 31) + 1024 + (threadIdx.x & ~31)];
      c = sm[(c & 31) + 2048 + (threadIdx.x & ~31)];
      d = sm[(d & 31) + 3072 + (threadIdx.x & ~31)];
    }
    if (MODE & 2) {
      e = __shfl_xor_sync(0xffffffffu, e, 1) + 1;
      f = __shfl_xor_sync(0xffffffffu, f, 2) + 1;
      g2 = __shfl_xor_sync(0xffffffffu, g2, 4) + 1;
      h = __shfl_xor_sync(0xffffffffu, h, 8) + 1;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d + e + f + g2 + h;
}
template <int MODE>
float run(int iters, int* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<MODE><<<148 * 4, 512>>>(iters, out);
  cudaEventRecord(e0);
  kern<MODE><<<148 * 4, 512>>>(iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}
int main() {
  int* out; cudaMalloc(&out, 148 * 4 * 512 * 4);
  const int it = 20000;
  float l = run<1>(it, out), s = run<2>(it, out), ls = run<3>(it, out);
  // per SM: 4 CTAs x 16 warps x it x 4 instructions
  double warp_instr = 4.0 * 16 * it * 4;
  double clk = 1.965e6;  // cycles per ms
  printf("LDS only %.3f ms (%.2f warp-LDS/clk/SM)  SHFL only %.3f ms (%.2f warp-SHFL/clk/SM)  both %.3f ms\n",
         l, warp_instr / (l * clk), s, warp_instr / (s * clk), ls);
  printf(ls < 0.8 * (l + s) ? "=> separate pipes (both ~ max)\n" : "=> shared pipe (both ~ sum)\n");
  return 0;
}
