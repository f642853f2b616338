// Launch-overhead micro-benchmark (latency mode): effective clock64 rate of a spinning
// CTA, and the event-timed cost of empty 1-CTA / 16-CTA / clustered (2 x 8) launches,
// back to back in a CUDA graph (as the single-pair align issues them).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch_overhead launch_overhead.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void spin(long long cycles, long long* out) {
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
  if (threadIdx.x == 0) out[0] = clock64() - t0;
}
__global__ void empty_k() {}
__global__ void __cluster_dims__(8, 1, 1) cluster_k() {
  cooperative_groups::this_cluster().sync();
}

template <typename F>
float graph_time(F launch, int reps) {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < reps; ++i) launch(s);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, s);
  cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / reps;  // us per launch
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  for (long long cyc : {1000000LL, 4000000LL}) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    spin<<<1, 32>>>(cyc, d);
    cudaEventRecord(a);
    spin<<<1, 32>>>(cyc, d);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("spin %lld cycles: %.1f us -> %.0f MHz effective clock64 rate\n", cyc, ms * 1e3,
           cyc / (ms * 1e3));
  }
  printf("empty 1-CTA launch in a graph: %.2f us\n",
         graph_time([](cudaStream_t s) { empty_k<<<1, 256, 0, s>>>(); }, 200));
  printf("empty 16-CTA launch in a graph: %.2f us\n",
         graph_time([](cudaStream_t s) { empty_k<<<16, 256, 0, s>>>(); }, 200));
  printf("clustered 2x8 CTAs + cluster sync in a graph: %.2f us\n",
         graph_time([](cudaStream_t s) { cluster_k<<<16, 256, 0, s>>>(); }, 200));
  printf("empty 1440-CTA launch in a graph: %.2f us\n",
         graph_time([](cudaStream_t s) { empty_k<<<1440, 128, 0, s>>>(); }, 200));
  return 0;
}
