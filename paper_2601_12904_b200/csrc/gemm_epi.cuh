// Fused GEMM epilogues shared by the 1-CTA and 2-CTA tcgen05 GEMMs: one call
// handles 32 consecutive fp32 accumulator columns of one output row (the
// registers of one tcgen05.ld 32x32b.x32).
#pragma once
#include "kernels.h"
#include "ptx.cuh"

namespace fragk {
namespace {

__device__ __forceinline__ float silu(float g) { return g / (1.0f + __expf(-g)); }

template <int EPI>
__device__ __forceinline__ void epi_chunk(const EpiParams& ep, int row, int col, const uint32_t (&r)[32],
                                          const uint32_t (&r2)[32]) {
  if constexpr (EPI == EPI_STORE_BF16) {
    uint4* dst = reinterpret_cast<uint4*>(ep.out_bf16 + (size_t)row * ep.ldo + col);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint4 v;
      v.x = pack_bf16(__uint_as_float(r[8 * j + 0]), __uint_as_float(r[8 * j + 1]));
      v.y = pack_bf16(__uint_as_float(r[8 * j + 2]), __uint_as_float(r[8 * j + 3]));
      v.z = pack_bf16(__uint_as_float(r[8 * j + 4]), __uint_as_float(r[8 * j + 5]));
      v.w = pack_bf16(__uint_as_float(r[8 * j + 6]), __uint_as_float(r[8 * j + 7]));
      dst[j] = v;
    }
  } else if constexpr (EPI == EPI_STORE_F32) {
    float4* dst = reinterpret_cast<float4*>(ep.out_f32 + (size_t)row * ep.ldo + col);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      dst[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]), __uint_as_float(r[4 * j + 2]),
                           __uint_as_float(r[4 * j + 3]));
  } else if constexpr (EPI == EPI_RESID) {
    float4* dst = reinterpret_cast<float4*>(ep.resid + (size_t)row * ep.ldo + col);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float4 h = dst[j];
      h.x += __uint_as_float(r[4 * j]);
      h.y += __uint_as_float(r[4 * j + 1]);
      h.z += __uint_as_float(r[4 * j + 2]);
      h.w += __uint_as_float(r[4 * j + 3]);
      dst[j] = h;
    }
  } else if constexpr (EPI == EPI_SWIGLU) {
    // col is the gate chunk's first column; the chunk is 64-aligned: gate block
    // (col/64) covers output columns [(col/64)*32, +32).
    uint4* dst = reinterpret_cast<uint4*>(ep.out_bf16 + (size_t)row * ep.ldo + (col >> 1));
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float a[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        float g = __uint_as_float(r[8 * j + t]);
        float u = __uint_as_float(r2[8 * j + t]);
        a[t] = silu(g) * u;
      }
      uint4 v;
      v.x = pack_bf16(a[0], a[1]);
      v.y = pack_bf16(a[2], a[3]);
      v.z = pack_bf16(a[4], a[5]);
      v.w = pack_bf16(a[6], a[7]);
      dst[j] = v;
    }
  } else if constexpr (EPI == EPI_QKV) {
    const int dh = ep.dh;
    const int q_cols = ep.Hq * dh;
    const int k_cols = ep.Hkv * dh;
    const int prow = ep.rows[row];
    float o[32];
    if (col < q_cols + k_cols) {
      // RoPE, interleaved pairs: o0 = k0 c - k1 s, o1 = k1 c + k0 s
      const int d0 = col % dh;
      const float2* cs = ep.rope + (size_t)prow * (dh >> 1) + (d0 >> 1);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        float2 t = cs[j];
        float k0 = __uint_as_float(r[2 * j]), k1 = __uint_as_float(r[2 * j + 1]);
        o[2 * j] = __fmaf_rn(k0, t.x, -(k1 * t.y));
        o[2 * j + 1] = __fmaf_rn(k1, t.x, k0 * t.y);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) o[j] = __uint_as_float(r[j]);
    }
    bf16* dstp;
    if (col < q_cols) {
      dstp = ep.q_out + (size_t)row * q_cols + col;
      if (ep.q_out_f32) {
        float4* qf = reinterpret_cast<float4*>(ep.q_out_f32 + (size_t)row * q_cols + col);
#pragma unroll
        for (int j = 0; j < 8; ++j) qf[j] = make_float4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
      }
    } else if (col < q_cols + k_cols) {
      dstp = ep.k_cache + (size_t)prow * k_cols + (col - q_cols);
    } else {
      dstp = ep.v_cache + (size_t)prow * k_cols + (col - q_cols - k_cols);
    }
    uint4* dst = reinterpret_cast<uint4*>(dstp);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint4 v;
      v.x = pack_bf16(o[8 * j + 0], o[8 * j + 1]);
      v.y = pack_bf16(o[8 * j + 2], o[8 * j + 3]);
      v.z = pack_bf16(o[8 * j + 4], o[8 * j + 5]);
      v.w = pack_bf16(o[8 * j + 6], o[8 * j + 7]);
      dst[j] = v;
    }
  }
}

}  // namespace
}  // namespace fragk
