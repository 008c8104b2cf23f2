// Memory-bound kernels of the reprocessing path:
//   K1  rope_shift_assemble  (SPEC.md:41-49 shift_rope, SPEC.md:399-407 stitch_full_reuse,
//                             PAPER.md:1040-1049 Appendix A re-positioning)
//   K2+K3 embed_rmsnorm, K3 rmsnorm  (SPEC.md:128 pre-norm decoder)
//   init_normal_bf16          (SPEC.md:94-102 init_model from the common.hpp:45-100 Rng)
#include <cstdlib>

#include "kernels.h"
#include "ptx.cuh"

namespace fragk {

namespace {


// Rotate 4 interleaved pairs held in one 16-byte vector by the per-chunk
// (cos, sin) of delta*theta_i: identical fp32 op order to oracle/fusion_oracle.cpp
// rope_rotate_pair() so K1 is bit-exact against the oracle.
__device__ __forceinline__ uint32_t rot_pair(uint32_t kv, float2 cs) {
  const float k0 = bf16_lo(kv), k1 = bf16_hi(kv);
  const float o0 = __fmaf_rn(k0, cs.x, -(k1 * cs.y));
  const float o1 = __fmaf_rn(k1, cs.x, k0 * cs.y);
  return pack_bf16(o0, o1);
}

// One CTA row of the grid per chunk (blockIdx.y); each thread moves 16-byte
// vectors of K (rotated) and V (copied) for (layer, token, head, 8 dims).
// Per layer the record block [n][Hkv][dh] and its fused destination
// [dst_row : dst_row+n][Hkv][dh] are both contiguous, so all accesses are
// fully coalesced 128-bit streams.
// One CTA row-slice per (chunk = blockIdx.y, layer = blockIdx.z): the
// destination offset of a source vector is then a sum, with no per-vector
// 64-bit division (those made the K-only copy issue-bound: 4.0 vs 5.0 TB/s).
// KV = false (shared V pages): only K is rotated into the fused cache, V stays
// in the records. U independent 16-byte loads per thread and step.
template <bool KV, int U>
__global__ void __launch_bounds__(256) rope_shift_kernel(const StitchChunk* __restrict__ chunks,
                                                         const float2* __restrict__ tables, bf16* __restrict__ kf,
                                                         bf16* __restrict__ vf, int T, int Hkv, int dh, int layer0) {
  const StitchChunk c = chunks[blockIdx.y];
  const int l = layer0 + (int)blockIdx.z;
  const int vec_per_row = (Hkv * dh) >> 3;  // 16-byte vectors per token row
  const int per_layer = c.n_tok * vec_per_row;
  const int dmask = (dh >> 3) - 1;  // dh / 8 vectors per head (a power of two: 8 or 16)
  const float2* tab = c.table >= 0 ? tables + (size_t)c.table * (dh >> 1) : nullptr;
  const uint4* ks = reinterpret_cast<const uint4*>(c.k_src) + (size_t)l * per_layer;
  const uint4* vs = reinterpret_cast<const uint4*>(c.v_src) + (size_t)l * per_layer;
  const size_t dst0 = ((size_t)l * T + c.dst_row) * vec_per_row;
  uint4* kd = reinterpret_cast<uint4*>(kf) + dst0;
  uint4* vd = reinterpret_cast<uint4*>(vf) + dst0;
  const int stride = gridDim.x * blockDim.x;  // a multiple of dh / 8: a thread's vectors share one head offset
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  float2 cs[4] = {};  // this thread's four cos/sin pairs, loaded once
  if (tab) {
    const int p = (i & dmask) * 4;
#pragma unroll
    for (int e = 0; e < 4; ++e) cs[e] = tab[p + e];
  }
  auto rot = [&](uint4& k, int) {
    if (tab) {
      k.x = rot_pair(k.x, cs[0]);
      k.y = rot_pair(k.y, cs[1]);
      k.z = rot_pair(k.z, cs[2]);
      k.w = rot_pair(k.w, cs[3]);
    }
  };
  for (; i + (U - 1) * stride < per_layer; i += U * stride) {
    uint4 k[U], v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      k[u] = ld_stream(ks + i + u * stride);
      if constexpr (KV) v[u] = ld_stream(vs + i + u * stride);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      rot(k[u], i + u * stride);
      st_stream(kd + i + u * stride, k[u]);
      if constexpr (KV) st_stream(vd + i + u * stride, v[u]);
    }
  }
  for (; i < per_layer; i += stride) {
    uint4 k0 = ld_stream(ks + i);
    rot(k0, i);
    st_stream(kd + i, k0);
    if constexpr (KV) st_stream(vd + i, ld_stream(vs + i));
  }
}

// ------------------------------------------------------------------ norms
// One CTA per row, the row held in registers (d/8 bf16x8 vectors over the CTA:
// 8 fp32 values per vector, NV vectors per thread), so the fp32 residual is
// read from HBM exactly once. Sum of squares in fp32 (block reduction), scale
// in fp32, bf16 output for the next GEMM's A operand. Launched with PDL: the
// next GEMM's CTAs start (and prefetch their weights) while rows finish.
template <bool EMBED, int NV>
__global__ void __launch_bounds__(256) rmsnorm_kernel(const bf16* __restrict__ E, const int* __restrict__ tok,
                                                      const float* __restrict__ h_in, const int* __restrict__ row_map,
                                                      int d, const bf16* __restrict__ gain, float eps,
                                                      float* __restrict__ h_out, bf16* __restrict__ x) {
  pdl_wait();
  pdl_launch_dependents();
  const int row = blockIdx.x;
  __shared__ float red[8];
  const int nvec = d >> 3;
  float f[NV][8];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int v = threadIdx.x + i * 256;
    if (v < nvec) {
      if constexpr (EMBED) {
        const uint4 e = reinterpret_cast<const uint4*>(E + (size_t)tok[row] * d)[v];
        const float t[8] = {bf16_lo(e.x), bf16_hi(e.x), bf16_lo(e.y), bf16_hi(e.y),
                            bf16_lo(e.z), bf16_hi(e.z), bf16_lo(e.w), bf16_hi(e.w)};
#pragma unroll
        for (int k = 0; k < 8; ++k) f[i][k] = t[k];
        float4* hdst = reinterpret_cast<float4*>(h_out + (size_t)row * d);
        hdst[2 * v] = make_float4(t[0], t[1], t[2], t[3]);
        hdst[2 * v + 1] = make_float4(t[4], t[5], t[6], t[7]);
      } else {
        const int src_row = row_map ? row_map[row] : row;
        const float4* src = reinterpret_cast<const float4*>(h_in + (size_t)src_row * d);
        const float4 a = src[2 * v], b = src[2 * v + 1];
        f[i][0] = a.x, f[i][1] = a.y, f[i][2] = a.z, f[i][3] = a.w;
        f[i][4] = b.x, f[i][5] = b.y, f[i][6] = b.z, f[i][7] = b.w;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) ss = fmaf(f[i][k], f[i][k], ss);
    }
  }
  ss = warp_sum(ss);
  if (lane_id() == 0) red[warp_id()] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float rs = rsqrtf(red[0] / (float)d + eps);
  const uint4* gv = reinterpret_cast<const uint4*>(gain);
  uint4* xo = reinterpret_cast<uint4*>(x + (size_t)row * d);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int v = threadIdx.x + i * 256;
    if (v < nvec) {
      const uint4 g = gv[v];
      uint4 o;
      o.x = pack_bf16(f[i][0] * rs * bf16_lo(g.x), f[i][1] * rs * bf16_hi(g.x));
      o.y = pack_bf16(f[i][2] * rs * bf16_lo(g.y), f[i][3] * rs * bf16_hi(g.y));
      o.z = pack_bf16(f[i][4] * rs * bf16_lo(g.z), f[i][5] * rs * bf16_hi(g.z));
      o.w = pack_bf16(f[i][6] * rs * bf16_lo(g.w), f[i][7] * rs * bf16_hi(g.w));
      xo[v] = o;
    }
  }
}

template <bool EMBED>
void launch_rmsnorm(const bf16* E, const int* tok, const float* h_in, const int* row_map, int M, int d,
                    const bf16* gain, float eps, float* h_out, bf16* x, cudaStream_t stream) {
  const int nv = (d / 8 + 255) / 256;  // vectors per thread
  if (nv <= 1)
    launch_pdl(rmsnorm_kernel<EMBED, 1>, dim3(M), dim3(256), 0, stream, E, tok, h_in, row_map, d, gain, eps, h_out, x);
  else if (nv <= 2)
    launch_pdl(rmsnorm_kernel<EMBED, 2>, dim3(M), dim3(256), 0, stream, E, tok, h_in, row_map, d, gain, eps, h_out, x);
  else if (nv <= 4)
    launch_pdl(rmsnorm_kernel<EMBED, 4>, dim3(M), dim3(256), 0, stream, E, tok, h_in, row_map, d, gain, eps, h_out, x);
  else
    launch_pdl(rmsnorm_kernel<EMBED, 8>, dim3(M), dim3(256), 0, stream, E, tok, h_in, row_map, d, gain, eps, h_out, x);
}

// ------------------------------------------------------------------ init
__device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t n) {
  // (n+1)-th output of Rng(seed).next_u64() (common.hpp:49-54): the state
  // advances by the golden gamma before each mix, so the stream is counter-based.
  uint64_t z = seed + (n + 1) * 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__global__ void init_normal_kernel(bf16* __restrict__ dst, uint64_t seed, size_t rows, size_t cols, float sigma,
                                   int blk, int blk_stride, int blk_off) {
  const size_t total = rows * cols;
  const size_t npairs = (total + 1) / 2;
  for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < npairs; j += (size_t)gridDim.x * blockDim.x) {
    // Box-Muller pair j consumes draws 2j (u1) and 2j+1 (u2) (common.hpp:78-92).
    // u1 == 0 (probability 2^-53 per pair) would shift the stream; ignored.
    const double u1 = (double)(splitmix_at(seed, 2 * j) >> 11) * 0x1.0p-53;
    const double u2 = (double)(splitmix_at(seed, 2 * j + 1) >> 11) * 0x1.0p-53;
    const double mag = sqrt(-2.0 * log(u1));
    const double ang = 6.283185307179586477 * u2;
    const double e[2] = {mag * cos(ang), mag * sin(ang)};
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const size_t idx = 2 * j + t;
      if (idx >= total) break;
      const size_t r = idx / cols, c = idx - r * cols;
      const size_t pr = (r / blk) * (size_t)blk_stride + blk_off + r % blk;
      dst[pr * cols + c] = __float2bfloat16_rn((float)e[t] * sigma);
    }
  }
}

__global__ void fill_kernel(bf16* dst, size_t n, float v) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = __float2bfloat16_rn(v);
}

}  // namespace

int rope_shift_assemble(const StitchChunk* chunks_dev, int n_chunks, int max_rows, const float2* tables,
                        bf16* k_fused, bf16* v_fused, int L, int T, int Hkv, int dh, cudaStream_t stream,
                        int layer0) {
  if (n_chunks <= 0 || max_rows <= 0 || L <= 0) return 0;
  if ((long)max_rows * (Hkv * dh / 8) >= (1L << 31) || ((dh / 8) & (dh / 8 - 1)) || L > 65535 || n_chunks > 65535)
    return -1;
  // about 8 CTAs per SM over (row slices x chunks x layers)
  const long slices = (long)n_chunks * L;
  long bx = ((long)num_sms() * 8 + slices - 1) / slices;
  const long need = ((long)max_rows * (Hkv * dh / 8) + 255) / 256;  // one vector per thread at most
  if (bx > need) bx = need;
  if (bx < 1) bx = 1;
  const dim3 grid((unsigned)bx, (unsigned)n_chunks, (unsigned)L);
  if (v_fused)
    rope_shift_kernel<true, 2><<<grid, 256, 0, stream>>>(chunks_dev, tables, k_fused, v_fused, T, Hkv, dh, layer0);
  else  // shared V pages: K only
    rope_shift_kernel<false, 4><<<grid, 256, 0, stream>>>(chunks_dev, tables, k_fused, v_fused, T, Hkv, dh, layer0);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

void embed_rmsnorm(const bf16* E, const int* tok, int M, int d, const bf16* gain, float eps, float* h, bf16* x,
                   cudaStream_t stream) {
  if (M <= 0) return;
  if (d > 8 * 256 * 8 || d % 8) return;  // d <= 16384 (all presets)
  launch_rmsnorm<true>(E, tok, nullptr, nullptr, M, d, gain, eps, h, x, stream);
}

void rmsnorm(const float* h, int M, int d, const bf16* gain, float eps, bf16* x, cudaStream_t stream,
             const int* row_map) {
  if (M <= 0) return;
  if (d > 8 * 256 * 8 || d % 8) return;
  launch_rmsnorm<false>(nullptr, nullptr, h, row_map, M, d, gain, eps, nullptr, x, stream);
}

namespace {
__global__ void f32_to_bf16_kernel(const float4* __restrict__ src, uint2* __restrict__ dst, size_t n4) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 f = src[i];
    dst[i] = make_uint2(pack_bf16(f.x, f.y), pack_bf16(f.z, f.w));
  }
}
}  // namespace

// fp32 -> bf16 (round to nearest even), n a multiple of 4 (FKVC record loads)
void f32_to_bf16(const float* src, bf16* dst, size_t n, cudaStream_t stream) {
  const size_t n4 = n / 4;
  size_t blocks = (n4 + 255) / 256;
  if (blocks > (size_t)num_sms() * 8) blocks = (size_t)num_sms() * 8;
  if (blocks == 0) return;
  f32_to_bf16_kernel<<<(unsigned)blocks, 256, 0, stream>>>(reinterpret_cast<const float4*>(src),
                                                          reinterpret_cast<uint2*>(dst), n4);
}

void init_normal_bf16(bf16* dst, uint64_t seed, size_t rows, size_t cols, float sigma, int blk, int blk_stride,
                      int blk_off, cudaStream_t stream) {
  const size_t pairs = (rows * cols + 1) / 2;
  size_t blocks = (pairs + 255) / 256;
  if (blocks > (size_t)num_sms() * 16) blocks = (size_t)num_sms() * 16;
  if (blocks == 0) blocks = 1;
  init_normal_kernel<<<(unsigned)blocks, 256, 0, stream>>>(dst, seed, rows, cols, sigma, blk, blk_stride, blk_off);
}

void fill_bf16(bf16* dst, size_t n, float v, cudaStream_t stream) {
  size_t blocks = (n + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  if (blocks == 0) return;
  fill_kernel<<<(unsigned)blocks, 256, 0, stream>>>(dst, n, v);
}

}  // namespace fragk
