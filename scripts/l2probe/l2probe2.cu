// L2 probe 2: random 8-byte gathers from a 48 MB buffer while the same
// threads stream a 2 GB array (12 B per gather, as a C5 column-block pass
// reads its matrix): streaming with __ldcs (ld.global.cs) vs plain loads vs
// no streaming. nvcc -O3 -gencode arch=compute_100a,code=sm_100a l2probe2.cu -o l2probe2
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull; z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull; z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
template <int Mode>  // 0 no stream, 1 __ldcs stream, 2 plain stream
__global__ void k(const double* __restrict__ x, int64_t n, const double* __restrict__ sv, const int* __restrict__ sc,
                  int64_t per_thread, double* out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, T = (int64_t)gridDim.x * blockDim.x;
  uint64_t st = mix(t);
  double acc = 0.0;
  for (int64_t i = 0; i < per_thread; ++i) {
    const int64_t e = i * T + t;  // coalesced stream position
    double v = 1.0;
    uint64_t c;
    if (Mode == 1) { v = __ldcs(sv + e); c = (uint64_t)(unsigned)__ldcs(sc + e); }
    else if (Mode == 2) { v = sv[e]; c = (uint64_t)(unsigned)sc[e]; }
    else c = 0;
    st = mix(st ^ c);
    acc = fma(v, __ldg(x + (int64_t)(st % (uint64_t)n)), acc);
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  const int64_t n = 48ll * (1 << 20) / 8;
  const int64_t ne = 160ll << 20;  // 160 M entries: 1.28 GB values + 0.64 GB columns
  double *x, *sv, *o; int* sc;
  cudaMalloc(&x, n * 8); cudaMemset(x, 0, n * 8);
  cudaMalloc(&sv, ne * 8); cudaMemset(sv, 0, ne * 8);
  cudaMalloc(&sc, ne * 4); cudaMemset(sc, 0, ne * 4);
  cudaMalloc(&o, 8);
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 8, block = 256;
  const int64_t per = ne / ((int64_t)grid * block);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 3; ++mode) {
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(a);
      if (mode == 0) k<0><<<grid, block>>>(x, n, sv, sc, per, o);
      if (mode == 1) k<1><<<grid, block>>>(x, n, sv, sc, per, o);
      if (mode == 2) k<2><<<grid, block>>>(x, n, sv, sc, per, o);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms = 0; cudaEventElapsedTime(&ms, a, b);
      const double g = (double)grid * block * per;
      if (r) printf("mode %d (%s): %.3f ms, %.1f Ggathers/s, stream %.0f GB/s\n", mode,
                    mode == 0 ? "gathers only" : mode == 1 ? "+ __ldcs stream" : "+ plain stream", ms,
                    g / (ms * 1e-3) / 1e9, mode ? g * 12 / (ms * 1e-3) / 1e9 : 0.0);
    }
  }
  return 0;
}
