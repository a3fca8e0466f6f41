// TMA gather4 probe: random rows of a 2D view of an L2-resident vector fetched
// by cp.async.bulk.tensor.2d...tile::gather4 (four arbitrary rows of W doubles
// per request, into shared memory) against the LSU gathers of l2probe.cu
// (~225 G 8-byte gathers/s: one L1TEX wavefront each). Question: does the TMA
// path, which bypasses L1TEX, fetch random 8-byte entries faster?
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tmagather.cu -o tmagather -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull; z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull; z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint32_t sptr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sptr(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, int bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sptr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, int phase) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(sptr(b)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int r0, int r1, int r2,
                                        int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
      "%6}], [%7];" ::"r"(sptr(dst)),
      "l"(tm), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(sptr(bar))
      : "memory");
}

// Each producer warp (lane 0) owns a ring of D stages; a stage = G gather4
// requests (4 rows x W doubles each) on one mbarrier.
template <int W, int G, int D>
__global__ void probe(const __grid_constant__ CUtensorMap tm, int64_t rows, int stages, double* out) {
  constexpr int kSlot = (4 * W + 15) / 16 * 16;  // doubles per request (128-B aligned)
  constexpr int kStage = G * kSlot;  // doubles per stage
  extern __shared__ __align__(1024) double smem[];
  __shared__ uint64_t bars[32][D];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* ring = smem + static_cast<size_t>(warp) * D * kStage;
  if (lane == 0)
    for (int d = 0; d < D; ++d) mbar_init(&bars[warp][d], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  uint64_t st = mix(blockIdx.x * 64ull + warp);
  double acc = 0.0;
  if (lane == 0) {
    for (int s = 0; s < stages + D; ++s) {
      const int d = s % D;
      if (s >= D) {  // retire stage s - D
        mbar_wait(&bars[warp][d], ((s - D) / D) & 1);
        acc += ring[d * kStage];
      }
      if (s < stages) {
        mbar_expect(&bars[warp][d], G * 4 * W * 8);
        for (int g = 0; g < G; ++g) {
          int r[4];
          for (int k = 0; k < 4; ++k) {
            st = mix(st);
            r[k] = static_cast<int>(__umul64hi(st, static_cast<uint64_t>(rows)));
          }
          gather4(ring + d * kStage + g * kSlot, &tm, &bars[warp][d], 0, r[0], r[1], r[2], r[3]);
        }
      }
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int W, int G, int D>
void run(EncodeFn enc, double* x, int64_t n, int sms, int warps, int ctas_per_sm) {
  const int64_t rows = n / W;
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)W * 8};
  cuuint32_t box[2] = {(cuuint32_t)W, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode W=%d failed %d\n", W, (int)r); return; }
  const size_t sm = static_cast<size_t>(warps) * D * G * ((4 * W + 15) / 16 * 16) * 8;
  cudaFuncSetAttribute(probe<W, G, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  double* o; cudaMalloc(&o, 8);
  const int grid = sms * ctas_per_sm, stages = 512;
  probe<W, G, D><<<grid, warps * 32, sm>>>(tm, rows, stages, o);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("W=%d launch: %s\n", W, cudaGetErrorString(e)); return; }
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) probe<W, G, D><<<grid, warps * 32, sm>>>(tm, rows, stages, o);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms = 0; cudaEventElapsedTime(&ms, a, b);
  const double reqs = 5.0 * grid * warps * stages * G;
  printf("W=%d doubles/row G=%d D=%d warps=%d ctas/SM=%d smem=%zu: %.1f G gather4/s = %.1f G rows/s, %.0f GB/s into smem\n",
         W, G, D, warps, ctas_per_sm, sm, reqs / (ms * 1e-3) / 1e9, 4 * reqs / (ms * 1e-3) / 1e9,
         4 * reqs * W * 8 / (ms * 1e-3) / 1e9);
  cudaFree(o);
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  EncodeFn enc = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  if (!enc) { printf("no encode fn\n"); return 1; }
  const int64_t n = 48ll * (1 << 20) / 8;
  double* x; cudaMalloc(&x, n * 8); cudaMemset(x, 0, n * 8);
  for (int warps : {1, 4, 8, 16, 32})
    for (int cps : {1, 2}) run<2, 4, 8>(enc, x, n, sms, warps, cps);
  run<2, 8, 8>(enc, x, n, sms, 4, 2);
  run<2, 4, 16>(enc, x, n, sms, 4, 2);
  run<4, 4, 8>(enc, x, n, sms, 4, 2);
  run<1, 4, 8>(enc, x, n, sms, 4, 2);
  return 0;
}
