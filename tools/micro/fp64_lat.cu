// FP64 dependent-chain latency and throughput vs ILP at 16 warps/SM (one
// 512-thread CTA per SM, as k_tdist runs), plus MUFU.RCP64H latency.
#include <cstdio>
#include <cuda_runtime.h>

template <int NCH>
__global__ void chains(int iters, double seed, double* out, long long* clk) {
  double x[NCH];
#pragma unroll
  for (int u = 0; u < NCH; ++u) x[u] = 1.0 + seed * (threadIdx.x + u);
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < NCH; ++u) x[u] = fma(x[u], 0.9999999, 1e-9);
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int u = 0; u < NCH; ++u) s += x[u];
  if (s == 12345.0) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) clk[0] = t1 - t0;
}

__global__ void mufu_lat(int iters, double seed, double* out, long long* clk) {
  double x = 1.5 + seed * threadIdx.x;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double r;
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    x = r;
  }
  const long long t1 = clock64();
  if (x == 12345.0) out[0] = x;
  if (threadIdx.x == 0 && blockIdx.x == 0) clk[0] = t1 - t0;
}

int main() {
  double* out;
  long long* clk;
  cudaMalloc(&out, 8);
  cudaMallocManaged(&clk, 8);
  const int iters = 8192;
  // latency: one warp
  chains<1><<<1, 32>>>(iters, 1e-7, out, clk);
  cudaDeviceSynchronize();
  chains<1><<<1, 32>>>(iters, 1e-7, out, clk);
  cudaDeviceSynchronize();
  printf("DFMA dependent latency: %.2f clk\n", (double)clk[0] / iters);
  mufu_lat<<<1, 32>>>(iters, 1e-7, out, clk);
  cudaDeviceSynchronize();
  mufu_lat<<<1, 32>>>(iters, 1e-7, out, clk);
  cudaDeviceSynchronize();
  printf("MUFU.RCP64H dependent latency: %.2f clk\n", (double)clk[0] / iters);
  // throughput at 16 warps/SM
  for (int nch : {1, 2, 4, 8, 16}) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (nch) {
        case 1: chains<1><<<148, 512>>>(iters, 1e-7, out, clk); break;
        case 2: chains<2><<<148, 512>>>(iters, 1e-7, out, clk); break;
        case 4: chains<4><<<148, 512>>>(iters, 1e-7, out, clk); break;
        case 8: chains<8><<<148, 512>>>(iters, 1e-7, out, clk); break;
        case 16: chains<16><<<148, 512>>>(iters, 1e-7, out, clk); break;
      }
      cudaDeviceSynchronize();
    }
    const double ops = (double)iters * nch * 512;  // per SM
    printf("16 warps/SM, %2d chains/thread: %.1f DFMA/clk/SM\n", nch, ops / clk[0]);
  }
  return 0;
}
