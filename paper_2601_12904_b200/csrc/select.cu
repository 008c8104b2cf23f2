// K9 qg_score + K10 topk_plan: query-guided critical-token selection
// (§3.2).
//
//   score[j] = sum_{t<Q} sum_{h<Hq} softmax_{j' in chunks}( q_{t,h} . k_{j,kv(h)} / sqrt(dh) )[j]
//
// The softmax is joint over all chunk keys of one (t, h), system
// and question keys are excluded, heads are summed, and the
// budget is a global top-k with lower-index tie-break.
//
// The scoring passes run on the tensor cores (score_tc.cu: exact three-term
// bf16 split of the fp32 queries); this file holds the row-statistics merge,
// the top-k plan (K10), the kv_deviation kernel of the CacheBlend selector and
// the greedy-decode argmax. No atomics on values: bit-deterministic.
#include <cfloat>

#include "kernels.h"
#include "ptx.cuh"

namespace fragk {

namespace {

// (max, sumexp) partials of the key groups -> (max, 1/Z) per (token, head) row
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

// Single-CTA top-k select + QIndexPlan. Each of the 32 warps owns a contiguous
// segment of the chunk keys and walks it 32 keys at a time (coalesced), so
// index order is kept with ballots instead of per-thread serial ranges:
//   1. 4 x 8-bit radix passes over order-preserving keys find the k-th largest
//      key tau and how many keys equal to tau are still needed (histogram with
//      leader-aggregated shared atomics: one request's scores share their
//      leading key bytes; match.any measured far slower);
//   2. per-warp counts of keys > tau and == tau, one warp-scan over the 32
//      warps -> each warp's output offset and its share of the tau ties (the
//      lowest indices win, SPEC.md:391 / SPEC.md:454);
//   3. ballot compaction in index order: plan_rows / plan_tok of the critical
//      rows, then the question rows.
template <bool STAGED>
__global__ void __launch_bounds__(TK_THREADS) topk_plan_kernel(const float* __restrict__ scores, int n, int k,
                                                                int key_row0, const int* __restrict__ chunk_tok,
                                                                const int* __restrict__ q_tok, int nq, int q_row0,
                                                                int* __restrict__ plan_rows,
                                                                int* __restrict__ plan_tok) {
  constexpr int NW = TK_THREADS / 32;
  __shared__ int hist[256];
  __shared__ int w_gt[NW], w_eq[NW];
  __shared__ uint32_t s_prefix;
  __shared__ int s_remaining;
  extern __shared__ uint32_t s_keys[];  // order-preserving keys of all scores (when they fit)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int seg = ((n + NW * 32 - 1) / (NW * 32)) * 32;  // per-warp segment, whole rounds
  const int w_lo = warp * seg, w_hi = min(n, w_lo + seg);
  if (STAGED) {
#pragma unroll 4
    for (int i = tid; i < n; i += TK_THREADS) s_keys[i] = fkey(scores[i]);
    __syncthreads();
  }
  auto key_at = [&](int i) { return STAGED ? s_keys[i] : fkey(scores[i]); };
  const bool all = k >= n;

  uint32_t tau = 0xFFFFFFFFu;
  int need_eq = 0;
  if (k > 0 && !all) {
    if (tid == 0) {
      s_prefix = 0;
      s_remaining = k;
    }
    uint32_t mask = 0;
    for (int shift = 24; shift >= 0; shift -= 8) {
      if (tid < 256) hist[tid] = 0;
      __syncthreads();
      const uint32_t prefix = s_prefix;
      for (int base = w_lo; base < w_hi; base += 32) {
        const int i = base + lane;
        const uint32_t key = i < w_hi ? key_at(i) : 0u;
        const bool hit = i < w_hi && (key & mask) == prefix;
        const int bin = hit ? (int)((key >> shift) & 255) : -1;
        // the first hit lane's bin takes one aggregated atomic (most keys of a
        // request share their leading bytes); the other lanes add their own
        const unsigned hits = __ballot_sync(0xffffffffu, hit);
        const int b0 = __shfl_sync(0xffffffffu, bin, hits ? __ffs(hits) - 1 : 0);
        const unsigned same = __ballot_sync(0xffffffffu, hit && bin == b0);
        if (hit) {
          if (bin != b0)
            atomicAdd(&hist[bin], 1);
          else if (lane == __ffs(same) - 1)
            atomicAdd(&hist[bin], __popc(same));
        }
      }
      __syncthreads();
      if (warp == 0) {
        // the bin holding the rem-th largest key: lane l scans bins 255-8l ..
        // 248-8l (descending); a warp scan gives each lane the count above them
        const int rem = s_remaining;
        int cnt[8], tot = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) tot += (cnt[e] = hist[255 - (lane * 8 + e)]);
        int incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        const int excl = incl - tot;
        const unsigned hit = __ballot_sync(0xffffffffu, excl < rem && rem <= incl);
        const int src = hit ? __ffs(hit) - 1 : 31;
        if (lane == src) {
          int cum = excl, b = 255 - lane * 8;
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            b = 255 - (lane * 8 + e);
            if (cum + cnt[e] >= rem || b == 0) break;
            cum += cnt[e];
          }
          s_remaining = rem - cum;
          s_prefix = prefix | ((uint32_t)b << shift);
        }
      }
      mask |= 255u << shift;
      __syncthreads();
    }
    tau = s_prefix;
    need_eq = s_remaining;
  }
  // per-warp counts of keys > tau and == tau
  int n_gt = 0, n_eq = 0;
  if (k > 0 && !all) {
    for (int base = w_lo; base < w_hi; base += 32) {
      const int i = base + lane;
      const uint32_t key = i < w_hi ? key_at(i) : 0u;
      n_gt += __popc(__ballot_sync(0xffffffffu, i < w_hi && key > tau));
      n_eq += __popc(__ballot_sync(0xffffffffu, i < w_hi && key == tau));
    }
  } else if (all) {
    n_gt = max(w_hi - w_lo, 0);
  }
  if (lane == 0) w_gt[warp] = n_gt, w_eq[warp] = n_eq;
  __syncthreads();
  // every warp scans the 32 warp totals: ties go to the lowest indices
  int take_eq = 0, out = 0;
  {
    const int g = w_gt[lane], e = w_eq[lane];
    int eq_in = e;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, eq_in, o);
      if (lane >= o) eq_in += y;
    }
    const int take_l = min(max(need_eq - (eq_in - e), 0), e);
    const int sel_l = g + take_l;
    int sel_in = sel_l;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, sel_in, o);
      if (lane >= o) sel_in += y;
    }
    take_eq = __shfl_sync(0xffffffffu, take_l, warp);
    out = __shfl_sync(0xffffffffu, sel_in - sel_l, warp);
  }
  // ballot compaction in index order
  if (k > 0) {
    int eq_seen = 0;
    for (int base = w_lo; base < w_hi; base += 32) {
      const int i = base + lane;
      const bool valid = i < w_hi;
      bool sel;
      if (all) {
        sel = valid;
      } else {
        const uint32_t key = valid ? key_at(i) : 0u;
        const bool eq = valid && key == tau;
        const unsigned eqm = __ballot_sync(0xffffffffu, eq);
        sel = (valid && key > tau) || (eq && eq_seen + __popc(eqm & lt) < take_eq);
        eq_seen += __popc(eqm);
      }
      const unsigned sm = __ballot_sync(0xffffffffu, sel);
      if (sel) {
        const int o = out + __popc(sm & lt);
        plan_rows[o] = key_row0 + i;
        plan_tok[o] = chunk_tok[i];
      }
      out += __popc(sm);
    }
  }
  // question rows follow the critical rows (they are the last positions)
  for (int i = tid; i < nq; i += TK_THREADS) {
    plan_rows[k + i] = q_row0 + i;
    plan_tok[k + i] = q_tok[i];
  }
}

}  // namespace

int score_combine(const ScoreArgs& a, int nblk, cudaStream_t stream) {
  score_combine_kernel<<<(a.nq * a.Hq + 255) / 256, 256, 0, stream>>>(a, nblk);
  return 1;
}

int qg_score(const ScoreArgs& a, cudaStream_t stream) { return qg_score_tc(a, stream); }

int topk_plan(const float* scores, int n_keys, int k, int key_row0, const int* chunk_tok, const int* q_tok, int nq,
              int q_row0, int* plan_rows, int* plan_tok, cudaStream_t stream) {
  const int smem = n_keys * (int)sizeof(uint32_t);
  if (smem <= 200 * 1024) {
    smem_attr_once(topk_plan_kernel<true>, 200 * 1024);
    topk_plan_kernel<true><<<1, TK_THREADS, smem, stream>>>(scores, n_keys, k, key_row0, chunk_tok, q_tok, nq,
                                                            q_row0, plan_rows, plan_tok);
  } else {  // > 51200 chunk tokens: every pass reads the scores from L2
    topk_plan_kernel<false><<<1, TK_THREADS, 0, stream>>>(scores, n_keys, k, key_row0, chunk_tok, q_tok, nq,
                                                          q_row0, plan_rows, plan_tok);
  }
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
