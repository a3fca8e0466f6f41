// Streaming-ceiling microbenchmark for the slab kernel's copy structure
// (timing experiment, not part of the library): a persistent grid whose
// producer warp bulk-copies fixed-size chunks of a buffer into `stages`
// shared-memory stages (mbarrier complete_tx) while consumer warps only
// release them, against a plain LDG.128 grid-stride read. Sweeping the buffer
// size separates bandwidth (slope) from per-launch overhead (intercept).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/sb scripts/stream_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t sm32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(288) tma_stream(const char* buf, long long bytes, int chunk, int stages,
                                                   int consumers, double* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[8], empty[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0)
    for (int q = 0; q < stages; ++q) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sm32(&full[q])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm32(&empty[q])), "r"(consumers));
    }
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncthreads();
  const long long nchunks = bytes / chunk;
  const long long per = (nchunks + gridDim.x - 1) / gridDim.x;
  const long long c0 = blockIdx.x * per, c1 = c0 + per < nchunks ? c0 + per : nchunks;
  if (warp == consumers) {
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      int i = 0;
      for (long long c = c0; c < c1; ++c, ++i) {
        const int st = i % stages;
        if (i >= stages) {
          const uint32_t ph = (i / stages - 1) & 1;
          asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(
                           sm32(&empty[st])), "r"(ph) : "memory");
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm32(&full[st])), "r"(chunk) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                sm32(sm + static_cast<size_t>(st) * chunk)),
            "l"(buf + c * chunk), "r"(chunk), "r"(sm32(&full[st])), "l"(pol)
            : "memory");
      }
    }
    return;
  }
  double acc = 0.0;
  int i = 0;
  for (long long c = c0; c < c1; ++c, ++i) {
    const int st = i % stages;
    const uint32_t ph = (i / stages) & 1;
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(
                     sm32(&full[st])), "r"(ph) : "memory");
    acc += reinterpret_cast<const double*>(sm + static_cast<size_t>(st) * chunk)[threadIdx.x];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sm32(&empty[st])) : "memory");
  }
  if (acc == 12345.678) sink[0] = acc;
}

__global__ void ldg_stream(const double2* buf, long long n4, double* sink) {
  double acc = 0.0;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  for (; i + 3 * stride < n4; i += 4 * stride) {
    double2 a = __ldcs(buf + i), b = __ldcs(buf + i + stride), c = __ldcs(buf + i + 2 * stride),
            d = __ldcs(buf + i + 3 * stride);
    acc += a.x + b.y + c.x + d.y;
  }
  for (; i < n4; i += stride) acc += __ldcs(buf + i).x;
  if (acc == 12345.678) sink[0] = acc;
}

int main() {
  const long long maxb = 432ll << 20;
  char* buf;
  double* sink;
  CK(cudaMalloc(&buf, maxb));
  CK(cudaMemset(buf, 0, maxb));
  CK(cudaMalloc(&sink, 8));
  char* flush;
  CK(cudaMalloc(&flush, 256 << 20));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  CK(cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  const long long sizes[3] = {54ll << 20, 108ll << 20, 432ll << 20};
  struct Cfg { int chunk, stages, cps; };
  const Cfg cfgs[] = {{28672, 3, 2}, {16384, 6, 2}, {32768, 3, 2}, {49152, 2, 2}, {24576, 4, 2},
                      {65536, 3, 1}, {32768, 6, 1}, {16384, 4, 3}, {8192, 8, 3}};
  for (const Cfg& c : cfgs) {
    const int grid = sms * c.cps;
    for (long long b : sizes) {
      float best = 1e9f;
      for (int rep = 0; rep < 3; ++rep) {
        CK(cudaMemsetAsync(flush, rep, 256 << 20));
        cudaEventRecord(e0);
        for (int k = 0; k < 10; ++k)
          tma_stream<<<grid, 288, c.chunk * c.stages>>>(buf, b, c.chunk, c.stages, 8, sink);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms / 10 < best ? ms / 10 : best;
      }
      CK(cudaGetLastError());
      printf("tma chunk %6d stages %d ctas/sm %d  %4lld MB: %8.2f us  %7.0f GB/s\n", c.chunk, c.stages, c.cps,
             b >> 20, best * 1e3, b / (best * 1e-3) / 1e9);
    }
  }
  for (int bs : {256, 512, 1024}) {
    for (int mult : {2, 4, 8}) {
      for (long long b : sizes) {
        float best = 1e9f;
        for (int rep = 0; rep < 3; ++rep) {
          cudaEventRecord(e0);
          for (int k = 0; k < 10; ++k) ldg_stream<<<sms * mult * 1024 / bs / 2, bs>>>(reinterpret_cast<const double2*>(buf), b / 16, sink);
          cudaEventRecord(e1);
          CK(cudaEventSynchronize(e1));
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          best = ms / 10 < best ? ms / 10 : best;
        }
        printf("ldg block %4d grid %5d  %4lld MB: %8.2f us  %7.0f GB/s\n", bs, sms * mult * 1024 / bs / 2, b >> 20,
               best * 1e3, b / (best * 1e-3) / 1e9);
      }
    }
  }
  return 0;
}
