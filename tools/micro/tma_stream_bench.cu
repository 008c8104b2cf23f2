// Microbenchmark: HBM read bandwidth of the weight-streaming access pattern
// (TMA 2D boxes of a K-major [N][K] bf16 matrix into a shared-memory ring,
// one CTA per SM, consumer releases each stage at once). Variants:
//   1: box 64 cols x 128 rows (128 B per row per request), 10 x 16 KB stages
//   2: two boxes adjacent in K per stage (256 B per row), 5 x 32 KB stages
//   3: box 64 cols x 256 rows, 5 x 32 KB stages
//   4: four boxes adjacent in K per stage (512 B per row), 3 x 64 KB stages
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_stream_bench tma_stream_bench.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}"
                 : "=r"(ok)
                 : "r"(su(b)), "r"(par)
                 : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
               ::"r"(su(dst)), "l"((uint64_t)m), "r"(su(bar)), "r"(x), "r"(y)
               : "memory");
}

template <int BOXES, int ROWS, int STAGES>
__global__ void __launch_bounds__(64, 1) stream(const __grid_constant__ CUtensorMap tm, int N, int K) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr uint32_t BOX = ROWS * 64 * 2, STAGE = BOX * BOXES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int tiles = N / ROWS, kst = K / (64 * BOXES);
  int stage = 0;
  uint32_t ph = 0;
  if (warp == 0 && lane == 0) {
    for (int t = blockIdx.x; t < tiles; t += gridDim.x)
      for (int k = 0; k < kst; ++k) {
        mbar_wait(&empty[stage], ph ^ 1);
        mbar_expect(&full[stage], STAGE);
        for (int b = 0; b < BOXES; ++b)
          tma2d(smem + stage * STAGE + b * BOX, &tm, &full[stage], (k * BOXES + b) * 64, t * ROWS);
        if (++stage == STAGES) stage = 0, ph ^= 1;
      }
  } else if (warp == 1 && lane == 0) {
    for (int t = blockIdx.x; t < tiles; t += gridDim.x)
      for (int k = 0; k < kst; ++k) {
        mbar_wait(&full[stage], ph);
        mbar_arrive(&empty[stage]);
        if (++stage == STAGES) stage = 0, ph ^= 1;
      }
  }
}

int main() {
  const int N = 28672, K = 4096;
  void* w;
  cudaMalloc(&w, (size_t)N * K * 2);
  cudaMemset(w, 0, (size_t)N * K * 2);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto run = [&](auto kern, int rows, size_t smem, const char* name) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)N};
    cuuint64_t str[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)rows};
    cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) kern<<<sms, 64, smem>>>(tm, N, K);
    cudaEventRecord(a);
    const int reps = 20;
    for (int i = 0; i < reps; ++i) kern<<<sms, 64, smem>>>(tm, N, K);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double gbs = (double)N * K * 2 * reps / (ms / 1e3) / 1e9;
    printf("%-40s %7.1f us  %7.1f GB/s  (%s)\n", name, ms * 1e3 / reps, gbs, cudaGetErrorString(cudaGetLastError()));
  };
  run(stream<1, 128, 10>, 128, 10 * 16384 + 1024, "1 box 128 rows x 128 B, 10 stages");
  run(stream<2, 128, 5>, 128, 5 * 32768 + 1024, "2 boxes (256 B per row), 5 stages");
  run(stream<1, 256, 5>, 256, 5 * 32768 + 1024, "1 box 256 rows x 128 B, 5 stages");
  run(stream<4, 128, 3>, 128, 3 * 65536 + 1024, "4 boxes (512 B per row), 3 stages");
  run(stream<2, 128, 6>, 128, 6 * 32768 + 1024, "2 boxes (256 B per row), 6 stages");
  return 0;
}
