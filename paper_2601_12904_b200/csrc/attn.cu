// K6 dispatch + split-KV combine for the sparse-Q attention (attn_tc.cu holds
// the tcgen05 kernel). SPEC.md:153-161.
#include <cfloat>

#include "kernels.h"
#include "ptx.cuh"

namespace fragk {

namespace {


// Merge split partials: out = sum_s w_s O_s / sum_s w_s, w_s = exp(lse_s - max).
// One warp per (token, head) row: the split weights are computed lane-parallel
// (one split per lane), then every lane accumulates DH/32 columns over the
// splits with coalesced loads, four splits in flight.
template <int DH>
__global__ void __launch_bounds__(128) attn_combine_kernel(const AttnArgs a) {
  constexpr int V = DH / 32;  // columns per lane
  pdl_wait();
  pdl_launch_dependents();
  const size_t MH = (size_t)a.M * a.Hq;
  const size_t qi = (size_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (qi >= MH) return;
  const int lane = threadIdx.x & 31;
  const int S = a.n_splits;
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
  const float* base = a.part_o + qi * DH + lane * V;
  for (int s0 = 0; s0 < S; s0 += 4) {
    float v[4][V];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int sp = s0 + u;
#pragma unroll
      for (int e = 0; e < V; ++e) v[u][e] = 0.f;
      if (sp < S) {
        if constexpr (V == 4) {
          const float4 t = __ldcg(reinterpret_cast<const float4*>(base + sp * MH * DH));
          v[u][0] = t.x, v[u][1] = t.y, v[u][2] = t.z, v[u][3] = t.w;
        } else {
          const float2 t = __ldcg(reinterpret_cast<const float2*>(base + sp * MH * DH));
          v[u][0] = t.x, v[u][1] = t.y;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int sp = s0 + u;
      const float w = __shfl_sync(0xffffffffu, sp < 32 ? wl[0] : wl[1], sp & 31);
      if (sp < S)
#pragma unroll
        for (int e = 0; e < V; ++e) acc[e] += w * v[u][e];
    }
  }
  const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
  bf16* out = a.out + qi * DH + lane * V;
#pragma unroll
  for (int e = 0; e < V; e += 2) *reinterpret_cast<uint32_t*>(out + e) = pack_bf16(acc[e] * inv, acc[e + 1] * inv);
}

}  // namespace

int sparse_q_attention(const AttnArgs& a0, cudaStream_t stream) {
  AttnArgs a = a0;
  if (a.M <= 0) return 0;
  if (a.Hkv <= 0 || a.Hq % a.Hkv != 0) return -1;
  const int G = a.Hq / a.Hkv;
  if (128 % G != 0) return -1;
  if (a.dh != 64 && a.dh != 128) return -1;
  const int tok_per_cta = attn_rows_per_cta() / G;  // query rows per CTA = tokens x G heads
  const int n_qblocks = (a.M + tok_per_cta - 1) / tok_per_cta;
  if (a.split_keys <= 0 || a.n_splits <= 1) a.n_splits = 1;
  if (attn_tc_launch(a, G, n_qblocks, stream) < 0) return -1;
  if (a.n_splits == 1) return 1;
  if (a.n_splits > 64) return -1;  // combine holds two split weights per lane
  const unsigned blocks = (unsigned)(((size_t)a.M * a.Hq + 3) / 4);
  if (a.dh == 128)
    launch_pdl(attn_combine_kernel<128>, dim3(blocks), dim3(128), 0, stream, a);
  else
    launch_pdl(attn_combine_kernel<64>, dim3(blocks), dim3(128), 0, stream, a);
  return 2;
}

}  // namespace fragk
