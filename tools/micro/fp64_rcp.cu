// Throughput of the reciprocal variants used by the Student-t passes (B200):
// DFMA, MUFU.RCP64H (rcp.approx.ftz.f64), rcp + 1/2 Newton steps, and an
// fp32 MUFU seed + fp64 Newton.  8 independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rcp64h(double q) {
  double r;
  asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
  return r;
}

template <int MODE>
__global__ void k(int iters, double seed, double* out) {
  double x[8], acc[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    x[u] = 1.5 + seed * (threadIdx.x + u);
    acc[u] = 0.0;
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double q = x[u];
      double r;
      if (MODE == 0) r = fma(q, 0.999, 0.001);                       // 1 DFMA
      if (MODE == 1) r = rcp64h(q);                                   // MUFU only
      if (MODE == 2) { r = rcp64h(q); r = fma(r, fma(-q, r, 1.0), r); }  // MUFU + 2 DFMA
      if (MODE == 3) {                                               // fp32 seed + 2 newton
        float f = __frcp_rn((float)q);
        r = (double)f;
        double e = fma(-q, r, 1.0);
        r = fma(r, fma(e, e, e), r);
      }
      acc[u] += r;
      x[u] = q + 1e-9;
    }
  }
  double s = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) s += acc[u];
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4096, blocks = 148 * 4, threads = 512;
  const char* names[] = {"DFMA+DADD", "MUFU.RCP64H+DADD", "rcp_q (MUFU+2DFMA)+DADD", "f32 seed+cubic"};
  for (int m = 0; m < 4; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      switch (m) {
        case 0: k<0><<<blocks, threads>>>(iters, 1e-7, out); break;
        case 1: k<1><<<blocks, threads>>>(iters, 1e-7, out); break;
        case 2: k<2><<<blocks, threads>>>(iters, 1e-7, out); break;
        case 3: k<3><<<blocks, threads>>>(iters, 1e-7, out); break;
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double n = (double)iters * 8 * blocks * threads;
      if (rep) printf("%-28s %.3f ms  %.1f G rcp/s  (%.2f warp-instr-slots/clk/SM per element)\n", names[m], ms,
                      n / ms / 1e6, n / 32 / (ms * 1e-3) / 148 / 1.965e9);
    }
  }
  return 0;
}
