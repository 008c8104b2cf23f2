// Split-KV combine of the sparse-Q attention (K6c), shared by the standalone
// combine kernel (attn.cu) and the GEMM chain's pre-op (gemm_chain.cu).
#pragma once
#include "kernels.h"
#include "ptx.cuh"

namespace fragk {

// Merge split partials: out = sum_s w_s O_s / sum_s w_s, w_s = exp(lse_s - max).
// One warp per (token, head) row qi: the split weights are computed
// lane-parallel (one split per lane), then every lane accumulates DH/32
// columns over the splits with coalesced loads.
template <int DH>
__device__ __forceinline__ void attn_combine_ld(const float* p, float (&v)[DH / 32]) {
  if constexpr (DH / 32 == 4) {
    const float4 t = __ldcg(reinterpret_cast<const float4*>(p));
    v[0] = t.x, v[1] = t.y, v[2] = t.z, v[3] = t.w;
  } else {
    const float2 t = __ldcg(reinterpret_cast<const float2*>(p));
    v[0] = t.x, v[1] = t.y;
  }
}

// Latency-bound (a handful of rows per warp, ~17 splits): the first batch of
// partial O loads is issued together with the split LSE loads, and the next
// batch is in flight while the current one is accumulated (batches of 8
// splits, accumulated in split order -> deterministic).
template <int DH>
__device__ __forceinline__ void attn_combine_row(const AttnArgs& a, size_t qi, int lane) {
  constexpr int V = DH / 32;  // columns per lane
  constexpr int B = 8;        // splits per batch
  const size_t MH = (size_t)a.M * a.Hq;
  const int S = a.n_splits;
  const float* base = a.part_o + qi * DH + lane * V;
  float cur[B][V], nxt[B][V];
#pragma unroll
  for (int u = 0; u < B; ++u) {
#pragma unroll
    for (int e = 0; e < V; ++e) cur[u][e] = 0.f;
    if (u < S) attn_combine_ld<DH>(base + u * MH * DH, cur[u]);
  }
  float wl[2] = {0.f, 0.f};  // weights of splits lane and lane + 32 (S <= 64)
  float mx = -INFINITY;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int sp = lane + 32 * h;
    wl[h] = sp < S ? a.part_lse[sp * MH + qi] : -INFINITY;
    mx = fmaxf(mx, wl[h]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float wsum = 0.f;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    wl[h] = (wl[h] == -INFINITY) ? 0.f : __expf(wl[h] - mx);
    wsum += wl[h];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
  float acc[V];
#pragma unroll
  for (int e = 0; e < V; ++e) acc[e] = 0.f;
  for (int s0 = 0; s0 < S; s0 += B) {
#pragma unroll
    for (int u = 0; u < B; ++u) {  // next batch in flight
#pragma unroll
      for (int e = 0; e < V; ++e) nxt[u][e] = 0.f;
      if (s0 + B + u < S) attn_combine_ld<DH>(base + (s0 + B + u) * MH * DH, nxt[u]);
    }
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int sp = s0 + u;
      const float w = __shfl_sync(0xffffffffu, sp < 32 ? wl[0] : wl[1], sp & 31);
      if (sp < S)
#pragma unroll
        for (int e = 0; e < V; ++e) acc[e] += w * cur[u][e];
    }
#pragma unroll
    for (int u = 0; u < B; ++u)
#pragma unroll
      for (int e = 0; e < V; ++e) cur[u][e] = nxt[u][e];
  }
  const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
  bf16* out = a.out + qi * DH + lane * V;
#pragma unroll
  for (int e = 0; e < V; e += 2) *reinterpret_cast<uint32_t*>(out + e) = pack_bf16(acc[e] * inv, acc[e + 1] * inv);
}

// Two rows per warp, their loads interleaved (the GEMM chain's pre-op: every
// warp owns ~2 rows, so the rows' dependent load rounds overlap). Same math
// and summation order per row as attn_combine_row.
template <int DH>
__device__ __forceinline__ void attn_combine_row2(const AttnArgs& a, size_t qa, size_t qb, bool has_b, int lane) {
  constexpr int V = DH / 32;
  constexpr int B = 8;
  const size_t MH = (size_t)a.M * a.Hq;
  const int S = a.n_splits;
  const size_t qi[2] = {qa, qb};
  const int nr = has_b ? 2 : 1;
  float cur[2][B][V];
  float wl[2][2], wsum[2];
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const float* base = a.part_o + qi[rr] * DH + lane * V;
#pragma unroll
    for (int u = 0; u < B; ++u) {
#pragma unroll
      for (int e = 0; e < V; ++e) cur[rr][u][e] = 0.f;
      if (rr < nr && u < S) attn_combine_ld<DH>(base + u * MH * DH, cur[rr][u]);
    }
  }
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    float mx = -INFINITY;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int sp = lane + 32 * h;
      wl[rr][h] = (rr < nr && sp < S) ? a.part_lse[sp * MH + qi[rr]] : -INFINITY;
      mx = fmaxf(mx, wl[rr][h]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float ws = 0.f;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      wl[rr][h] = (wl[rr][h] == -INFINITY) ? 0.f : __expf(wl[rr][h] - mx);
      ws += wl[rr][h];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ws += __shfl_xor_sync(0xffffffffu, ws, o);
    wsum[rr] = ws;
  }
  float acc[2][V];
#pragma unroll
  for (int rr = 0; rr < 2; ++rr)
#pragma unroll
    for (int e = 0; e < V; ++e) acc[rr][e] = 0.f;
  for (int s0 = 0; s0 < S; s0 += B) {
#pragma unroll
    for (int rr = 0; rr < 2; ++rr)
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int sp = s0 + u;
        const float w = __shfl_sync(0xffffffffu, sp < 32 ? wl[rr][0] : wl[rr][1], sp & 31);
        if (sp < S)
#pragma unroll
          for (int e = 0; e < V; ++e) acc[rr][e] += w * cur[rr][u][e];
      }
    if (s0 + B < S) {
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        const float* base = a.part_o + qi[rr] * DH + lane * V;
#pragma unroll
        for (int u = 0; u < B; ++u) {
#pragma unroll
          for (int e = 0; e < V; ++e) cur[rr][u][e] = 0.f;
          if (rr < nr && s0 + B + u < S) attn_combine_ld<DH>(base + (s0 + B + u) * MH * DH, cur[rr][u]);
        }
      }
    }
  }
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    if (rr >= nr) break;
    const float inv = wsum[rr] > 0.f ? 1.f / wsum[rr] : 0.f;
    bf16* out = a.out + qi[rr] * DH + lane * V;
#pragma unroll
    for (int e = 0; e < V; e += 2)
      *reinterpret_cast<uint32_t*>(out + e) = pack_bf16(acc[rr][e] * inv, acc[rr][e + 1] * inv);
  }
}

}  // namespace fragk
