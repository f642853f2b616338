// Microbenchmark: cost of one fixed-order reduction of 1-2 doubles over
// (a) a 256/512-thread CTA, (b) + an 8-CTA cluster via barrier + DSMEM,
// (c) + an 8-CTA cluster via remote-store + flag polling (no barrier).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

template <int NT>
__device__ double block_sum(double v, double* scr, int& par) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
  double* s = scr + par * 32; par ^= 1;
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
  __syncthreads();
  v = (threadIdx.x & 31) < NT / 32 ? s[threadIdx.x & 31] : 0.0;
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
  return v;
}

template <int NT, int MODE>
__global__ void k(int iters, double* out, long long* cyc) {
  __shared__ double scr[64];
  __shared__ double cb[2][8];
  __shared__ volatile unsigned flag[2][8];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank();
  if (threadIdx.x < 16) { ((double*)cb)[threadIdx.x] = 0; flag[threadIdx.x/8][threadIdx.x%8] = 0; }
  cl.sync();
  int par = 0;
  double v = threadIdx.x * 1e-3 + rank;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    double s = block_sum<NT>(v, scr, par);
    if (MODE == 1) {
      const int p = it & 1;
      if (threadIdx.x == 0) cb[p][rank] = s;
      cl.sync();
      double t = 0;
#pragma unroll
      for (int r = 0; r < 8; ++r) t += cl.map_shared_rank(&cb[p][0], r)[rank];  // dummy pattern
      s = t;
    } else if (MODE == 2) {
      const int p = it & 1;
      if (threadIdx.x < 8) {  // push my partial + seq to every rank
        double* rc = cl.map_shared_rank(&cb[p][0], threadIdx.x);
        rc[rank] = s;
        asm volatile("fence.acq_rel.cluster;" ::: "memory");
        volatile unsigned* rf = (volatile unsigned*)cl.map_shared_rank((unsigned*)&flag[p][0], threadIdx.x);
        rf[rank] = it + 1;
      }
      if (threadIdx.x < 8) { while (flag[p][threadIdx.x] != (unsigned)(it + 1)) {} }
      __syncwarp();
      asm volatile("fence.acq_rel.cluster;" ::: "memory");
      __syncthreads();
      double t = 0;
#pragma unroll
      for (int r = 0; r < 8; ++r) t += ((volatile double*)cb[p])[r];
      s = t;
    }
    v = s * 1e-9 + v;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && rank == 0) { out[blockIdx.x] = v; cyc[0] = (t1 - t0) / iters; }
  cl.sync();
}

template <int NT, int MODE>
void run(const char* name) {
  double* out; long long* cyc; cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 8);
  cudaLaunchConfig_t c = {}; c.gridDim = dim3(8); c.blockDim = dim3(NT);
  cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = 8; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
  c.attrs = a; c.numAttrs = 1;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2000;
  cudaLaunchKernelEx(&c, k<NT, MODE>, iters, out, cyc);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&c, k<NT, MODE>, iters, out, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-34s %7.3f us/reduction  %6lld cycles  (%s)\n", name, ms * 1e3 / iters, h,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<256, 0>("block only, 256 thr");
  run<512, 0>("block only, 512 thr");
  run<256, 1>("block + cluster barrier, 256 thr");
  run<512, 1>("block + cluster barrier, 512 thr");
  run<256, 2>("block + cluster flags, 256 thr");
  return 0;
}
