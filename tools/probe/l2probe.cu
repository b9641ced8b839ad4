// L2 residency probe: random 4-byte gathers into an array of S MB (indices from an
// in-kernel hash, no index stream), 2^27 gathers per launch.  Run under ncu with
// dram__bytes_read.sum to see the effective L2 capacity for random reads.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__global__ void gather(const int* __restrict__ a, long n, long iters, int* out) {
  unsigned long long x = (blockIdx.x * 1024ull + threadIdx.x) * 0x9E3779B97F4A7C15ull + 1;
  int acc = 0;
  for (long i = 0; i < iters; ++i) {
    x ^= x >> 12; x ^= x << 25; x ^= x >> 27;
    const long j = (long)((x * 0x2545F4914F6CDD1Dull) % (unsigned long long)n);
    acc += __ldg(a + j);
  }
  if (acc == 0x7fffffff) out[0] = acc;
}
int main(int argc, char** argv) {
  for (int ai = 1; ai < argc; ++ai) {
    const long mb = atol(argv[ai]);
    const long n = mb * (1l << 20) / 4;
    int* a; int* o;
    cudaMalloc(&a, n * 4); cudaMalloc(&o, 4);
    cudaMemset(a, 1, n * 4);
    const int blocks = 148 * 8, threads = 256;
    const long iters = (1l << 27) / (blocks * threads);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      gather<<<blocks, threads>>>(a, n, iters, o);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2) printf("%ld MB: %.3f ms, %.1f Ggathers/s\n", mb, ms, (double)blocks * threads * iters / ms / 1e6);
    }
    cudaFree(a); cudaFree(o);
  }
  return 0;
}
