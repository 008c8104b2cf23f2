// K9 qg_score + K10 topk_plan: query-guided critical-token selection
// (§3.2).
//
//   score[j] = sum_{t<Q} sum_{h<Hq} softmax_{j' in chunks}( q_{t,h} . k_{j,kv(h)} / sqrt(dh) )[j]
//
// The softmax is joint over all chunk keys of one (t, h), system
// and question keys are excluded, heads are summed, and the
// budget is a global top-k with lower-index tie-break.
//
// fp32 CUDA-core FMAs so scores follow the fp32 oracle to summation-order
// rounding; no atomics, so the result is bit-deterministic run to run.
#include <cfloat>

#include "kernels.h"
#include "ptx.cuh"

namespace fragk {

namespace {

constexpr int SC_KEYS = 64;     // keys per CTA
constexpr int SC_ROWS = 128;    // query rows per shared-memory tile
constexpr int SC_THREADS = 256;
constexpr int SC_PAD = 4;       // row padding (floats): conflict-free 128-bit shared loads

template <int DH>
constexpr size_t score_smem() { return (size_t)(SC_KEYS + SC_ROWS) * (DH + SC_PAD) * sizeof(float); }

// Register-tiled fp32 CUDA-core scoring: a CTA owns 64 keys and walks the kv
// heads and their query rows; each thread computes an 8-row x 4-key block
// with 128-bit shared-memory operand loads (12 loads per 128 FMAs). Every dot
// product is a sequential fp32 FMA chain over dh, exactly as in the fp32
// oracle restatement, and all reductions run in a fixed order (no atomics), so
// scores are bit-deterministic.
// MODE 1: per-(block,row) (max, sumexp) of scaled logits.
// MODE 2: column sums of softmax probabilities (row_ms = (max, 1/Z)).
// MODE 3: column sums of raw scaled logits.
template <int MODE, int DH>
__global__ void __launch_bounds__(SC_THREADS) score_kernel(const ScoreArgs a) {
  constexpr int LD = DH + SC_PAD;
  extern __shared__ float4 sc_smem4[];
  float* sk = reinterpret_cast<float*>(sc_smem4);  // [SC_KEYS][LD]
  float* sq = sk + SC_KEYS * LD;                   // [SC_ROWS][LD]
  __shared__ float colsum[SC_THREADS / 32][SC_KEYS];
  const int blk = blockIdx.x;
  const int key0 = blk * SC_KEYS;
  const int nrows_tot = a.nq * a.Hq;
  const int G = a.Hq / a.Hkv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // thread -> rows rg*8 .. rg*8+7 of the row tile, keys kg + 16*j (j < 4)
  const int rg = tid >> 4, kg = tid & 15;
  float csum[4] = {0.f, 0.f, 0.f, 0.f};

  for (int hk = 0; hk < a.Hkv; ++hk) {
    __syncthreads();
    for (int idx = tid; idx < SC_KEYS * (DH / 8); idx += SC_THREADS) {
      const int r = idx / (DH / 8), c8 = (idx % (DH / 8)) * 8;
      const int j = key0 + r;
      float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if (j < a.n_keys) {
        const uint4 u = *reinterpret_cast<const uint4*>(a.k + ((size_t)(a.key_row0 + j) * a.Hkv + hk) * DH + c8);
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          v[2 * e] = __uint_as_float(w[e] << 16);
          v[2 * e + 1] = __uint_as_float(w[e] & 0xffff0000u);
        }
      }
      float4* dst = reinterpret_cast<float4*>(sk + r * LD + c8);
      dst[0] = make_float4(v[0], v[1], v[2], v[3]);
      dst[1] = make_float4(v[4], v[5], v[6], v[7]);
    }
    const int nrows = a.nq * G;  // rows of this kv group: (t, g) -> row t*Hq + hk*G + g
    for (int r0 = 0; r0 < nrows; r0 += SC_ROWS) {
      __syncthreads();
      for (int idx = tid; idx < SC_ROWS * (DH / 4); idx += SC_THREADS) {
        const int r = idx / (DH / 4), c4 = (idx % (DH / 4)) * 4;
        const int rr = r0 + r;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (rr < nrows) {
          const int t = rr / G, g = rr % G;
          v = *reinterpret_cast<const float4*>(a.q + ((size_t)t * a.Hq + hk * G + g) * DH + c4);
        }
        *reinterpret_cast<float4*>(sq + r * LD + c4) = v;
      }
      __syncthreads();
      // both 8-row groups of this warp past the end (warp-uniform: the shuffles
      // below need the full warp; no barrier follows inside this iteration)
      if (r0 + (rg & ~1) * 8 >= nrows) continue;
      float acc[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
#pragma unroll 2
      for (int c = 0; c < DH; c += 4) {
        float4 kv[4], qv[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) kv[j] = *reinterpret_cast<const float4*>(sk + (kg + 16 * j) * LD + c);
#pragma unroll
        for (int i = 0; i < 8; ++i) qv[i] = *reinterpret_cast<const float4*>(sq + (rg * 8 + i) * LD + c);
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float t = fmaf(qv[i].x, kv[j].x, acc[i][j]);
            t = fmaf(qv[i].y, kv[j].y, t);
            t = fmaf(qv[i].z, kv[j].z, t);
            acc[i][j] = fmaf(qv[i].w, kv[j].w, t);
          }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int rr = r0 + rg * 8 + i;
        const bool rvalid = rr < nrows;
        const int grow = rvalid ? (rr / G) * a.Hq + hk * G + rr % G : 0;
        if constexpr (MODE == 1) {
          // local (max, sumexp) over this CTA's 64 keys for row grow: the 16 kg lanes
          float sv[4];
          float mx = -INFINITY;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const bool kvalid = key0 + kg + 16 * j < a.n_keys;
            sv[j] = kvalid ? acc[i][j] * a.scale : -INFINITY;
            mx = fmaxf(mx, sv[j]);
          }
#pragma unroll
          for (int o = 1; o < 16; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
          float z = 0.f;
#pragma unroll
          for (int j = 0; j < 4; ++j) z += (sv[j] == -INFINITY) ? 0.f : __expf(sv[j] - mx);
#pragma unroll
          for (int o = 1; o < 16; o <<= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
          if (kg == 0 && rvalid) a.part_ms[(size_t)blk * nrows_tot + grow] = make_float2(mx, z);
        } else if constexpr (MODE == 2) {
          if (rvalid) {
            const float2 ms = a.row_ms[grow];
#pragma unroll
            for (int j = 0; j < 4; ++j) csum[j] += __expf(acc[i][j] * a.scale - ms.x) * ms.y;
          }
        } else {
          if (rvalid) {
#pragma unroll
            for (int j = 0; j < 4; ++j) csum[j] += acc[i][j] * a.scale;
          }
        }
      }
    }
  }
  if constexpr (MODE != 1) {
    // deterministic column reduction: the two row groups of a warp, then the 8 warps in order
#pragma unroll
    for (int j = 0; j < 4; ++j) csum[j] += __shfl_xor_sync(0xffffffffu, csum[j], 16);
    if (lane < 16)
#pragma unroll
      for (int j = 0; j < 4; ++j) colsum[warp][kg + 16 * j] = csum[j];
    __syncthreads();
    if (tid < SC_KEYS) {
      float s = 0.f;
      for (int w = 0; w < SC_THREADS / 32; ++w) s += colsum[w][tid];
      const int j = key0 + tid;
      if (j < a.n_keys) a.scores[j] = s;
    }
  }
}

__global__ void score_combine_kernel(const ScoreArgs a, int nblk) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  const int nrows = a.nq * a.Hq;
  if (row >= nrows) return;
  float mx = -INFINITY;
  for (int b = 0; b < nblk; ++b) mx = fmaxf(mx, a.part_ms[(size_t)b * nrows + row].x);
  float z = 0.f;
  for (int b = 0; b < nblk; ++b) {
    const float2 p = a.part_ms[(size_t)b * nrows + row];
    if (p.x != -INFINITY) z += p.y * __expf(p.x - mx);
  }
  a.row_ms[row] = make_float2(mx, z > 0.f ? 1.f / z : 0.f);
}

// ---------------------------------------------------------------- K10
constexpr int TK_THREADS = 1024;

__device__ __forceinline__ uint32_t fkey(float f) {
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// Block-wide exclusive scan of one int per thread (1024 threads).
__device__ int block_excl_scan(int v, int* sh, int* total) {
  const int lane = lane_id(), w = warp_id();
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    int s = sh[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    sh[lane] = s;  // inclusive warp totals
  }
  __syncthreads();
  const int base = w > 0 ? sh[w - 1] : 0;
  if (total) *total = sh[31];
  __syncthreads();
  return base + x - v;
}

__global__ void __launch_bounds__(TK_THREADS) topk_plan_kernel(const float* __restrict__ scores, int n, int k,
                                                                int key_row0, const int* __restrict__ chunk_tok,
                                                                const int* __restrict__ q_tok, int nq, int q_row0,
                                                                int* __restrict__ plan_rows,
                                                                int* __restrict__ plan_tok) {
  __shared__ int hist[256];
  __shared__ int sh[32];
  __shared__ uint32_t s_prefix;
  __shared__ int s_remaining;
  const int tid = threadIdx.x;
  const int per = (n + TK_THREADS - 1) / TK_THREADS;
  const int lo = tid * per, hi = min(lo + per, n);

  uint32_t tau = 0xFFFFFFFFu;
  int need_eq = 0;
  if (k > 0 && k < n) {
    if (tid == 0) {
      s_prefix = 0;
      s_remaining = k;
    }
    uint32_t mask = 0;
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int b = tid; b < 256; b += TK_THREADS) hist[b] = 0;
      __syncthreads();
      const uint32_t prefix = s_prefix;
      for (int i = lo; i < hi; ++i) {
        const uint32_t key = fkey(scores[i]);
        if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1);
      }
      __syncthreads();
      if (tid == 0) {
        int rem = s_remaining, cum = 0, b = 255;
        for (; b > 0; --b) {
          if (cum + hist[b] >= rem) break;
          cum += hist[b];
        }
        s_remaining = rem - cum;
        s_prefix = prefix | ((uint32_t)b << shift);
      }
      mask |= 255u << shift;
      __syncthreads();
    }
    tau = s_prefix;
    need_eq = s_remaining;
  } else if (k >= n) {
    tau = 0;
    need_eq = n;  // everything selected (all keys >= 0 in key space)
  }
  // pass: count > tau and == tau in my range
  int n_gt = 0, n_eq = 0;
  if (k > 0) {
    for (int i = lo; i < hi; ++i) {
      const uint32_t key = fkey(scores[i]);
      if (k >= n) {
        ++n_gt;
      } else {
        n_gt += key > tau;
        n_eq += key == tau;
      }
    }
  }
  const int eq_before = block_excl_scan(n_eq, sh, nullptr);
  int take_eq = (k >= n) ? 0 : min(max(need_eq - eq_before, 0), n_eq);
  const int my_sel = n_gt + take_eq;
  int total = 0;
  int out = block_excl_scan(my_sel, sh, &total);
  if (k > 0) {
    int eq_seen = 0;
    for (int i = lo; i < hi; ++i) {
      bool sel;
      if (k >= n) {
        sel = true;
      } else {
        const uint32_t key = fkey(scores[i]);
        if (key > tau) sel = true;
        else if (key == tau) sel = (eq_seen++ < take_eq);
        else sel = false;
      }
      if (sel) {
        plan_rows[out] = key_row0 + i;
        plan_tok[out] = chunk_tok[i];
        ++out;
      }
    }
  }
  // question rows follow the critical rows (they are the last positions)
  for (int i = tid; i < nq; i += TK_THREADS) {
    plan_rows[k + i] = q_row0 + i;
    plan_tok[k + i] = q_tok[i];
  }
}

}  // namespace

template <int DH>
int qg_score_dh(const ScoreArgs& a, int nblk, cudaStream_t stream) {
  constexpr int SM = (int)score_smem<DH>();
  smem_attr_once(score_kernel<1, DH>, SM);
  smem_attr_once(score_kernel<2, DH>, SM);
  smem_attr_once(score_kernel<3, DH>, SM);
  if (!a.raw) {
    score_kernel<1, DH><<<nblk, SC_THREADS, SM, stream>>>(a);
    score_combine_kernel<<<(a.nq * a.Hq + 255) / 256, 256, 0, stream>>>(a, nblk);
    score_kernel<2, DH><<<nblk, SC_THREADS, SM, stream>>>(a);
    return 3;
  }
  score_kernel<3, DH><<<nblk, SC_THREADS, SM, stream>>>(a);
  return 1;
}

int qg_score(const ScoreArgs& a, cudaStream_t stream) {
  const int nblk = (a.n_keys + SC_KEYS - 1) / SC_KEYS;
  if (nblk <= 0) return 0;
  if (a.Hq % a.Hkv != 0) return -1;
  if (a.dh == 128) return qg_score_dh<128>(a, nblk, stream);
  if (a.dh == 64) return qg_score_dh<64>(a, nblk, stream);
  return -1;
}

int topk_plan(const float* scores, int n_keys, int k, int key_row0, const int* chunk_tok, const int* q_tok, int nq,
              int q_row0, int* plan_rows, int* plan_tok, cudaStream_t stream) {
  topk_plan_kernel<<<1, TK_THREADS, 0, stream>>>(scores, n_keys, k, key_row0, chunk_tok, q_tok, nq, q_row0,
                                                 plan_rows, plan_tok);
  return 1;
}

// ------------------------------------------------------------------ greedy step
// argmax over one logits row (lowest index on ties: the greedy decoding rule of
// SPEC.md:137 / 438); the winner is written to out[0] (or out[(*out_idx)++]) and,
// for the next decode step, to plan_tok[0] with plan_rows[0] = next_row
// (next_row < 0: plan_rows[0] + 1, so a captured step needs no host value).
namespace {
constexpr int AM_THREADS = 1024;
__global__ void __launch_bounds__(AM_THREADS) argmax_kernel(const float* __restrict__ logits, int V, int* out,
                                                            int* out_idx, int* plan_tok, int* plan_rows,
                                                            int next_row) {
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < V; i += AM_THREADS) {
    const float v = logits[i];
    if (v > best) best = v, bi = i;  // strided scan: first hit of a value is its lowest index here
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) best = ov, bi = oi;
  }
  __shared__ float sv[AM_THREADS / 32];
  __shared__ int si[AM_THREADS / 32];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sv[w] = best, si[w] = bi;
  __syncthreads();
  if (w == 0) {
    best = sv[l], bi = si[l];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) best = ov, bi = oi;
    }
    if (l == 0) {
      if (bi == 0x7fffffff) bi = 0;  // all-NaN row: token 0
      if (out_idx) {  // device-side slot counter: graph-replayable decode steps
        out[out_idx[0]] = bi;
        out_idx[0] += 1;
      } else {
        out[0] = bi;
      }
      if (plan_tok) plan_tok[0] = bi;
      if (plan_rows) plan_rows[0] = next_row >= 0 ? next_row : plan_rows[0] + 1;
    }
  }
}
}  // namespace

int greedy_argmax(const float* logits, int V, int* out, int* out_idx, int* plan_tok, int* plan_rows, int next_row,
                  cudaStream_t stream) {
  argmax_kernel<<<1, AM_THREADS, 0, stream>>>(logits, V, out, out_idx, plan_tok, plan_rows, next_row);
  return 1;
}

// ------------------------------------------------------------------ kv_deviation (Eq. 7)
// Delta_KV[j, l, c] = sum_{e < Hkv*dh} (KV_FA[l][j][e] - KV_FR[l][j][e])^2 for
// c = K, V. One warp per (token, layer):
// 128-bit loads of both caches (each row read once: HBM-bound), fp32 squared
// differences summed per lane in a fixed order, then a fixed butterfly -> bit-
// deterministic. The selection vector of select_cacheblend (SPEC.md:417-425,
// Eq. 8: Delta_KV[:, 2, 1]) is written for layer sel_layer from the same sums.
namespace {
constexpr int DV_WARPS = 8;
__device__ __forceinline__ float sq_diff8(const uint4 a, const uint4 b) {
  const __nv_bfloat162* pa = reinterpret_cast<const __nv_bfloat162*>(&a);
  const __nv_bfloat162* pb = reinterpret_cast<const __nv_bfloat162*>(&b);
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 fa = __bfloat1622float2(pa[i]);
    const float2 fb = __bfloat1622float2(pb[i]);
    const float d0 = fa.x - fb.x, d1 = fa.y - fb.y;
    acc = fmaf(d0, d0, acc);
    acc = fmaf(d1, d1, acc);
  }
  return acc;
}

__global__ void __launch_bounds__(DV_WARPS * 32) kv_deviation_kernel(const DeviationArgs a) {
  const int warp = blockIdx.x * DV_WARPS + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (warp >= a.n_rows * a.n_layers) return;
  const int j = warp / a.n_layers, l = warp % a.n_layers;
  const int nvec = a.width / 8;
  const uint4* ka = reinterpret_cast<const uint4*>(a.k_fa + (size_t)l * a.fa_layer_stride + (size_t)j * a.width);
  const uint4* va = reinterpret_cast<const uint4*>(a.v_fa + (size_t)l * a.fa_layer_stride + (size_t)j * a.width);
  const uint4* kb = reinterpret_cast<const uint4*>(a.k_fr + (size_t)l * a.fr_layer_stride + (size_t)j * a.width);
  const uint4* vb = reinterpret_cast<const uint4*>(a.v_fr + (size_t)l * a.fr_layer_stride + (size_t)j * a.width);
  float dk = 0.f, dv = 0.f;
  for (int i = lane; i < nvec; i += 32) {
    dk += sq_diff8(__ldcs(ka + i), __ldcs(kb + i));
    dv += sq_diff8(__ldcs(va + i), __ldcs(vb + i));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dk += __shfl_xor_sync(0xffffffffu, dk, o);
    dv += __shfl_xor_sync(0xffffffffu, dv, o);
  }
  if (lane == 0) {
    if (a.dev) {
      a.dev[((size_t)j * a.n_layers + l) * 2 + 0] = dk;
      a.dev[((size_t)j * a.n_layers + l) * 2 + 1] = dv;
    }
    if (a.sel_scores && l == a.sel_layer)
      a.sel_scores[j] = a.sel_comp == 0 ? dk : (a.sel_comp == 1 ? dv : dk + dv);
  }
}
}  // namespace

int kv_deviation(const DeviationArgs& a, cudaStream_t stream) {
  if (a.n_rows <= 0 || a.n_layers <= 0) return 0;
  if (a.width % 8 != 0) return -1;
  const long warps = (long)a.n_rows * a.n_layers;
  kv_deviation_kernel<<<(unsigned)((warps + DV_WARPS - 1) / DV_WARPS), DV_WARPS * 32, 0, stream>>>(a);
  return 1;
}

}  // namespace fragk
