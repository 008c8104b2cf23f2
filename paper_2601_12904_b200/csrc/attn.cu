// K6 dispatch + split-KV combine for the sparse-Q attention (attn_tc.cu holds
// the tcgen05 kernel). SPEC.md:153-161.
#include <cfloat>

#include "attn_combine.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace fragk {

namespace {


template <int DH>
__global__ void __launch_bounds__(128) attn_combine_kernel(const AttnArgs a) {
  pdl_wait();
  pdl_launch_dependents();
  const size_t qi = (size_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (qi >= (size_t)a.M * a.Hq) return;
  attn_combine_row<DH>(a, qi, threadIdx.x & 31);
}

}  // namespace

int sparse_q_attention(const AttnArgs& a0, cudaStream_t stream, bool* combine_deferred) {
  AttnArgs a = a0;
  if (combine_deferred) *combine_deferred = false;
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
  if (combine_deferred) {  // the caller runs the combine (GEMM chain pre-op)
    *combine_deferred = true;
    return 1;
  }
  const unsigned blocks = (unsigned)(((size_t)a.M * a.Hq + 3) / 4);
  if (a.dh == 128)
    launch_pdl(attn_combine_kernel<128>, dim3(blocks), dim3(128), 0, stream, a);
  else
    launch_pdl(attn_combine_kernel<64>, dim3(blocks), dim3(128), 0, stream, a);
  return 2;
}

}  // namespace fragk
