// Fused GEMM epilogues shared by the 1-CTA and 2-CTA tcgen05 GEMMs: one call
// handles 32 consecutive fp32 accumulator columns of one output row (the
// registers of one tcgen05.ld 32x32b.x32).
#pragma once
#include "kernels.h"
#include "ptx.cuh"

namespace fragk {
namespace {

__device__ __forceinline__ float silu(float g) { return g / (1.0f + __expf(-g)); }

// Folded RMSNorm scale of one row (1 unless the consumer reads partials):
// the producer's per-chunk Σh² summed in chunk order, four running sums.
template <int EPI>
__device__ __forceinline__ float epi_row_scale(const EpiParams& ep, int row) {
  if constexpr (EPI == EPI_QKV || EPI == EPI_SWIGLU) {
    if (ep.ssq_in) {
      const float* p = ep.ssq_in + row;
      const size_t ld = (size_t)ep.ssq_ld;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
      int i = 0;
      if (ep.l2_reads) {  // GEMM chain: written by other CTAs of the same launch
#pragma unroll 4
        for (; i + 4 <= ep.ssq_n; i += 4) {
          s0 += __ldcg(p + i * ld);
          s1 += __ldcg(p + (i + 1) * ld);
          s2 += __ldcg(p + (i + 2) * ld);
          s3 += __ldcg(p + (i + 3) * ld);
        }
      } else {
#pragma unroll 4
        for (; i + 4 <= ep.ssq_n; i += 4) {
          s0 += p[i * ld];
          s1 += p[(i + 1) * ld];
          s2 += p[(i + 2) * ld];
          s3 += p[(i + 3) * ld];
        }
      }
      for (; i < ep.ssq_n; ++i) s0 += __ldcg(p + i * ld);
      return rsqrtf(((s0 + s1) + (s2 + s3)) / (float)ep.norm_d + ep.norm_eps);
    }
  }
  return 1.f;
}

template <int EPI>
__device__ __forceinline__ void epi_chunk(const EpiParams& ep, int row, int col, const uint32_t (&r)[32],
                                          const uint32_t (&r2)[32], float rs = 1.f) {
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
    float4 hv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      // GEMM chain: an earlier op of the same launch may have written it on another SM
      float4 h = ep.l2_reads ? __ldcg(dst + j) : dst[j];
      h.x += __uint_as_float(r[4 * j]);
      h.y += __uint_as_float(r[4 * j + 1]);
      h.z += __uint_as_float(r[4 * j + 2]);
      h.w += __uint_as_float(r[4 * j + 3]);
      dst[j] = h;
      hv[j] = h;
    }
    if (ep.x_out) {
      float ss = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        ss = fmaf(hv[j].x, hv[j].x, ss);
        ss = fmaf(hv[j].y, hv[j].y, ss);
        ss = fmaf(hv[j].z, hv[j].z, ss);
        ss = fmaf(hv[j].w, hv[j].w, ss);
      }
      ep.ssq_out[(size_t)(col >> 5) * ep.ssq_ld + row] = ss;
      uint4* xo = reinterpret_cast<uint4*>(ep.x_out + (size_t)row * ep.ldo + col);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint4 v;
        v.x = pack_bf16(hv[2 * j].x, hv[2 * j].y);
        v.y = pack_bf16(hv[2 * j].z, hv[2 * j].w);
        v.z = pack_bf16(hv[2 * j + 1].x, hv[2 * j + 1].y);
        v.w = pack_bf16(hv[2 * j + 1].z, hv[2 * j + 1].w);
        xo[j] = v;
      }
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
        float g = __uint_as_float(r[8 * j + t]) * rs;
        float u = __uint_as_float(r2[8 * j + t]) * rs;
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
      const int ppos = ep.rows_per_seq > 0 ? prow % ep.rows_per_seq : prow;
      const float2* cs = ep.rope + (size_t)ppos * (dh >> 1) + (d0 >> 1);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        float2 t = cs[j];
        float k0 = __uint_as_float(r[2 * j]) * rs, k1 = __uint_as_float(r[2 * j + 1]) * rs;
        o[2 * j] = __fmaf_rn(k0, t.x, -(k1 * t.y));
        o[2 * j + 1] = __fmaf_rn(k1, t.x, k0 * t.y);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) o[j] = __uint_as_float(r[j]) * rs;
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
      const int vrow = !ep.v_slots ? prow : (prow >= ep.v_tail_row0 ? ep.v_tail_slot0 + (prow - ep.v_tail_row0) : row);
      dstp = ep.v_cache + (size_t)vrow * k_cols + (col - q_cols - k_cols);
    }
    uint4* dst = reinterpret_cast<uint4*>(dstp);
    uint4* dst2 = (ep.v_cache2 && col >= q_cols + k_cols)
                      ? reinterpret_cast<uint4*>(ep.v_cache2 + (size_t)prow * k_cols + (col - q_cols - k_cols))
                      : nullptr;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint4 v;
      v.x = pack_bf16(o[8 * j + 0], o[8 * j + 1]);
      v.y = pack_bf16(o[8 * j + 2], o[8 * j + 3]);
      v.z = pack_bf16(o[8 * j + 4], o[8 * j + 5]);
      v.w = pack_bf16(o[8 * j + 6], o[8 * j + 7]);
      dst[j] = v;
      if (dst2) dst2[j] = v;
    }
  }
}


// Sum n fp32 partials (row-major rows of BN, `sstride` floats apart) of this
// thread's row in partial order and run the fused epilogue on 32-column
// chunk units u = u0, u0 + du, ... (a unit is 2 chunks for SwiGLU); rs = the
// row's folded RMSNorm scale (epi_row_scale, loaded by the caller early).
template <int BN, int EPI>
__device__ __forceinline__ void reduce_partials(const EpiParams& ep, const float* base, size_t sstride, int n,
                                                int u0, int du, int row, int col0, float rs) {
  constexpr int CW = EPI == EPI_SWIGLU ? 2 : 1;
  constexpr int UNITS = BN / 32 / CW;
#pragma unroll 1
  for (int u = u0; u < UNITS; u += du) {
    uint32_t r[2][32];
#pragma unroll
    for (int h2 = 0; h2 < CW; ++h2) {
      const int c = u * CW + h2;
      float4 acc[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      int s2 = 0;
      for (; s2 + 1 < n; s2 += 2) {  // two partials in flight per step
        const float4* a = reinterpret_cast<const float4*>(base + s2 * sstride + c * 32);
        const float4* b = reinterpret_cast<const float4*>(base + (s2 + 1) * sstride + c * 32);
        float4 va[8], vb[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) va[j] = __ldcg(a + j), vb[j] = __ldcg(b + j);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          acc[j].x += va[j].x, acc[j].y += va[j].y, acc[j].z += va[j].z, acc[j].w += va[j].w;
          acc[j].x += vb[j].x, acc[j].y += vb[j].y, acc[j].z += vb[j].z, acc[j].w += vb[j].w;
        }
      }
      if (s2 < n) {
        const float4* a = reinterpret_cast<const float4*>(base + s2 * sstride + c * 32);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 v = __ldcg(a + j);
          acc[j].x += v.x, acc[j].y += v.y, acc[j].z += v.z, acc[j].w += v.w;
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        r[h2][4 * j] = __float_as_uint(acc[j].x);
        r[h2][4 * j + 1] = __float_as_uint(acc[j].y);
        r[h2][4 * j + 2] = __float_as_uint(acc[j].z);
        r[h2][4 * j + 3] = __float_as_uint(acc[j].w);
      }
    }
    epi_chunk<EPI>(ep, row, col0 + u * CW * 32, r[0], r[CW - 1], rs);
  }
}

// ---------------------------------------------------------------- split-K fixup
// Cooperative, deterministic reduction of one split-K tile slot. Every split
// CTA has written its fp32 partial (ws_rows x BN, row-major, one row per TMEM
// lane) to ep.ws slot (slot*S + sp). All S split CTAs of the slot are
// co-resident (persistent grid), so instead of one last-arriving CTA reducing
// the whole tile, each waits for all S partials and then reduces and runs the
// fused epilogue on its own share of the 32-column chunks (round-robin by
// split index), summing the partials in split order -> bit-identical results
// whatever the arrival order. Called by the 4 epilogue warps (128 threads,
// named barrier 1); `warp2_lane0` does the counter traffic.
template <int BN, int EPI>
__device__ __forceinline__ void split_fixup(const EpiParams& ep, int slot, int S, int sp, int ws_rows,
                                            int row_in_tile, int row, int M, int col0, bool warp2_lane0,
                                            float rs) {
  __threadfence();
  asm volatile("bar.sync 1, 128;" ::: "memory");
  int* cnt = ep.counters + slot;
  if (warp2_lane0) {
    atomicAdd(cnt, 1);
    spin_until_ge(cnt, S, ep.fault, ep.spin_ns, 64);
  }
  asm volatile("bar.sync 1, 128;" ::: "memory");
  const float* base = ep.ws + ((size_t)slot * S * ws_rows + row_in_tile) * BN;
  if (row_in_tile < ws_rows && row < M)
    reduce_partials<BN, EPI>(ep, base, (size_t)ws_rows * BN, S, sp, S, row, col0, rs);
  // second round of arrivals: the last CTA out resets the counter for the next GEMM
  asm volatile("bar.sync 1, 128;" ::: "memory");
  if (warp2_lane0) {
    const int old = atomicAdd(cnt, 1);
    if (old == 2 * S - 1) *cnt = 0;
  }
}

// ---------------------------------------------------------------- stream-K
// CTA whose k-block range [c*I/G, (c+1)*I/G) holds flattened k-block pos.
__device__ __forceinline__ int sk_cta_of(long long pos, long long I, int G) {
  int c = (int)(pos * G / I);
  while (c + 1 < G && I * (c + 1) / G <= pos) ++c;
  while (c > 0 && I * c / G > pos) --c;
  return c;
}

// Finish one stream-K part of a tile shared by n CTAs (this one is the j-th,
// counted from the owner; its partial is already in workspace slot j).
// Contributors (j > 0) publish and leave; the owner (j = 0, whose part is its
// last) waits for the n-1 others, sums slots 0..n-1 in order and runs the
// fused epilogue. 4 epilogue warps, named barrier 1.
template <int BN, int EPI>
__device__ __forceinline__ void sk_finish(const EpiParams& ep, int tile, int j, int n, int ws_rows, int row_in_tile,
                                          int row, int M, int col0, bool leader, float rs) {
  __threadfence();
  asm volatile("bar.sync 1, 128;" ::: "memory");
  int* cnt = ep.counters + tile;
  if (j > 0) {
    if (leader) atomicAdd(cnt, 1);
    return;
  }
  if (leader) {
    spin_until_ge(cnt, n - 1, ep.fault, ep.spin_ns);
    *cnt = 0;  // every contributor has arrived: reset for the next GEMM
  }
  asm volatile("bar.sync 1, 128;" ::: "memory");
  const float* base = ep.ws + ((size_t)tile * ep.sk_maxc * ws_rows + row_in_tile) * BN;
  if (row_in_tile < ws_rows && row < M)
    reduce_partials<BN, EPI>(ep, base, (size_t)ws_rows * BN, n, 0, 1, row, col0, rs);
}

}  // namespace
}  // namespace fragk
