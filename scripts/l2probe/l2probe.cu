// L2 probe: random 8-byte gathers from a buffer of S MB by every SM, against
// each half of the SMs (by %smid) gathering only from "its" half of the buffer.
// Question: does a B200 die keep its own copy of lines (effective L2 per die
// ~63 MB), so that die-local column blocks would hit where shared ones miss?
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a l2probe.cu -o l2probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smid() { unsigned s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s)); return s; }
__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull; z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull; z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
// mode 0: every CTA gathers over [0, n); mode 1: CTAs on SMs < split gather over
// [0, n/2), the others over [n/2, n)
__global__ void gather(const double* __restrict__ x, int64_t n, int iters, int mode, unsigned split, double* out) {
  const unsigned s = smid();
  int64_t lo = 0, len = n;
  if (mode == 1) { len = n / 2; lo = s < split ? 0 : n / 2; }
  uint64_t st = mix(blockIdx.x * 1024ull + threadIdx.x);
  double acc = 0.0;
  for (int i = 0; i < iters; ++i) {
    st = mix(st);
    acc += __ldg(x + lo + (int64_t)(st % (uint64_t)len));
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mb : {24, 40, 48, 64, 80, 96}) {
    const int64_t n = (int64_t)mb * (1 << 20) / 8;
    double* x; cudaMalloc(&x, n * 8); cudaMemset(x, 0, n * 8);
    double* o; cudaMalloc(&o, 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int grid = sms * 8, block = 256, iters = 256;
    for (int mode = 0; mode < 2; ++mode) {
      for (unsigned split : {74u}) {
        gather<<<grid, block>>>(x, n, iters, mode, split, o);  // warm
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) gather<<<grid, block>>>(x, n, iters, mode, split, o);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms = 0; cudaEventElapsedTime(&ms, a, b);
        const double g = 5.0 * grid * block * (double)iters;
        printf("%3d MB mode %d (split %u): %.3f ms, %.1f Ggathers/s\n", mb, mode, split, ms / 5, g / (ms * 1e-3) / 1e9);
      }
    }
    cudaFree(x); cudaFree(o);
  }
  return 0;
}
