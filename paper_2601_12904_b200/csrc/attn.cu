// K6 dispatch + split-KV combine for the sparse-Q attention (attn_tc.cu holds
// the tcgen05 kernel). SPEC.md:153-161.
#include <cfloat>

#include "kernels.h"
#include "ptx.cuh"

namespace fragk {

namespace {


// Merge split partials: out = sum_s w_s O_s / sum_s w_s, w_s = exp(lse_s - max).
template <int DH>
__global__ void attn_combine_kernel(const AttnArgs a) {
  const size_t qi = blockIdx.x;  // (token, head)
  const size_t MH = (size_t)a.M * a.Hq;
  float mx = -INFINITY;
  for (int s = 0; s < a.n_splits; ++s) mx = fmaxf(mx, a.part_lse[s * MH + qi]);
  const int d = threadIdx.x;  // DH threads
  float acc = 0.f, wsum = 0.f;
  for (int s = 0; s < a.n_splits; ++s) {
    const float lse = a.part_lse[s * MH + qi];
    if (lse == -INFINITY) continue;
    const float w = __expf(lse - mx);
    wsum += w;
    acc += w * a.part_o[(s * MH + qi) * DH + d];
  }
  a.out[qi * DH + d] = __float2bfloat16_rn(wsum > 0.f ? acc / wsum : 0.f);
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
  if (a.dh == 128)
    attn_combine_kernel<128><<<(unsigned)((size_t)a.M * a.Hq), 128, 0, stream>>>(a);
  else
    attn_combine_kernel<64><<<(unsigned)((size_t)a.M * a.Hq), 64, 0, stream>>>(a);
  return 2;
}

}  // namespace fragk
