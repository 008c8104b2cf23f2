// Microbenchmark: exp2 throughput on the SFU for fp32 vs packed f16x2 / bf16x2
// (elements per second), to size the attention softmax. nvcc -gencode arch=compute_100a,code=sm_100a
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

template <int MODE>
__global__ void k(float* out, int iters) {
  float a[8];
  uint32_t h[8];
  for (int i = 0; i < 8; ++i) {
    a[i] = -0.001f * (threadIdx.x + i);
    h[i] = 0xbc00bc00u + i;  // small negative halves
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      } else if (MODE == 1) {
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h[i]));
      } else if (MODE == 2) {
        asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h[i]));
      } else if (MODE == 3) {
        asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[i]));
      } else if (MODE == 4) {
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h[i]) : "f"(a[i]), "f"(__uint_as_float(h[i])));
      } else if (MODE == 6) {  // truncating pack: the high halves of two fp32 (one PRMT)
        asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(h[i]) : "r"(__float_as_uint(a[i])), "r"(h[(i + 1) & 7]));
      } else {  // softmax mix: 2 MUFU + 1 pack
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[(i + 1) & 7]));
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h[i]) : "f"(a[i]), "f"(a[(i + 1) & 7]));
      }
    }
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i] + __uint_as_float(h[i]);
  if (s == 123.f) out[0] = s;
}

int main(int argc, char** argv) {
  float* o;
  cudaMalloc(&o, 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096, threads = argc > 1 ? atoi(argv[1]) : 512, blocks = sms * (argc > 2 ? atoi(argv[2]) : 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[7] = {"ex2.f32", "ex2.f16x2", "ex2.bf16x2", "ffma.f32", "f2fp.pack", "2ex2+pack", "prmt.pack"};
  for (int m = 0; m < 7; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (m == 0) k<0><<<blocks, threads>>>(o, iters);
      if (m == 1) k<1><<<blocks, threads>>>(o, iters);
      if (m == 2) k<2><<<blocks, threads>>>(o, iters);
      if (m == 3) k<3><<<blocks, threads>>>(o, iters);
      if (m == 4) k<4><<<blocks, threads>>>(o, iters);
      if (m == 5) k<5><<<blocks, threads>>>(o, iters);
      if (m == 6) k<6><<<blocks, threads>>>(o, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double ops = (double)blocks * threads * iters * 8;  // instructions (lanes)
      const double elems = ops * (m == 1 || m == 2 || m == 5 ? 2 : 1);
      if (rep) printf("%-10s %8.3f ms  %7.2f Tinst/s  %7.2f Telem/s  per SM per clk (1.9GHz): %.1f elems\n", names[m], ms,
                      ops / ms / 1e9, elems / ms / 1e9, elems / (ms * 1e-3) / sms / 1.9e9);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
