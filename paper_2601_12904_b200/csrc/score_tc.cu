// K9 qg_score on the 5th-gen tensor cores (select_query_guided scoring,
// SPEC.md:426-434; §3.2):
//
//   score[j] = sum_{t<Q} sum_{h<Hq} softmax_{j' in chunks}( q_{t,h} . k_{j,kv(h)} / sqrt(dh) )[j]
//
// The question's final-layer queries stay fp32 (the selection is an index set
// that must agree with the fp32 oracle). Each fp32 query is
// split exactly into three bf16 terms q = q_hi + q_mid + q_lo (24 mantissa
// bits); keys are bf16 already, so every product q_i * k is exact in the fp32
// accumulator and S = sum_i Q_i K^T reproduces the fp32 dot product up to
// accumulation order (~1e-7 relative) -- three bf16 tcgen05.mma instead of an
// fp32 CUDA-core FMA chain, which is what made the old kernel ALU-bound.
//
// One CTA = one kv head x one 128-row query tile (rows (t, g) of that GQA
// group) x a contiguous group of 128-key blocks. 6 warps:
//   warps 0-3  one thread per TMEM lane
//   warp 4     TMA producer: the tile's three bf16 query terms (written by
//              score_split_kernel), then the kv head's 128-key K blocks
//              (SW128) into a 2-stage ring
//   warp 5     TMEM alloc (2 x 128 columns) + single-thread MMA issue
// Pass 1 (MODE 1): S = Q K^T (lanes = query rows): online (max, sumexp) per
//   row over the group's keys -> part_ms[group][row]; score_combine_kernel
//   (select.cu) merges the groups into (max, 1/Z).
// Pass 2 (MODE 2 softmax / MODE 3 raw logits): S^T = K Q^T (lanes = keys): each
//   thread sums its key's probabilities over the 128 rows in a fixed order ->
//   col_part[kv head, row tile][key]; score_head_sum_kernel adds the Hkv x
//   row-tile partials in a fixed order. No atomics anywhere: bit-deterministic.
#include <cuda.h>

#include <algorithm>
#include <cfloat>

#include "kernels.h"
#include "ptx.cuh"

namespace fragk {

namespace {

constexpr int ST_ROWS = 128;  // query rows per tile (TMEM lanes in pass 1)
constexpr int ST_KEYS = 128;  // keys per block (TMEM lanes in pass 2)
constexpr int ST_THREADS = 192;
constexpr int ST_SPLITS = 3;  // bf16 terms per fp32 query
constexpr float LOG2E = 1.4426950408889634f;

template <int DH>
struct ScoreCfg {
  static constexpr int ATOMS = DH / 64;
  static constexpr uint32_t Q_SPLIT = ST_ROWS * DH * 2;  // one bf16 term, [ATOMS][128][64]
  static constexpr uint32_t K_BYTES = ST_KEYS * DH * 2;  // one key block
  static constexpr int STAGES = DH == 128 ? 3 : 4;  // K ring depth
  static constexpr size_t SMEM =
      1024 + ST_SPLITS * (size_t)Q_SPLIT + STAGES * (size_t)K_BYTES + 2 * ST_ROWS * 4 + 256;
  static_assert(SMEM <= 232448, "score tile exceeds the 227 KB shared-memory limit");
};

// fp32 -> bf16 bits, round to nearest even (finite inputs)
__device__ __forceinline__ uint32_t bf16_bits(float x) {
  return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(x));
}
__device__ __forceinline__ float bf16_val(uint32_t b) { return __uint_as_float(b << 16); }

template <int MODE, int DH>
__global__ void __launch_bounds__(ST_THREADS, 1)
    score_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmQ,
                    const ScoreArgs a, int blocks_per_group, int r_pad) {
  using C = ScoreCfg<DH>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                           // [SPLITS][Q_SPLIT]
  uint8_t* sK = sQ + ST_SPLITS * C::Q_SPLIT;    // [STAGES][K_BYTES]
  float* s_m = reinterpret_cast<float*>(sK + C::STAGES * C::K_BYTES);  // pass 2: row max (natural units)
  float* s_w = s_m + ST_ROWS;                                  // pass 2: 1/Z (or 1 / 0 for raw)
  uint64_t* bar = reinterpret_cast<uint64_t*>(s_w + ST_ROWS);
  uint64_t* k_full = bar + 0;   // [4]
  uint64_t* k_empty = bar + 4;  // [4]
  uint64_t* s_full = bar + 8;   // [2]
  uint64_t* s_empty = bar + 10; // [2]
  uint64_t* q_ready = bar + 12;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 13);

  const int warp = warp_id(), lane = lane_id();
  const int grp = blockIdx.x, mt = blockIdx.y, hk = blockIdx.z;
  const int G = a.Hq / a.Hkv;
  const int R = a.nq * G;  // query rows of this kv head
  const int nrows_tot = a.nq * a.Hq;
  const int n_blocks = (a.n_keys + ST_KEYS - 1) / ST_KEYS;
  const int b_lo = grp * blocks_per_group;
  const int b_hi = min(b_lo + blocks_per_group, n_blocks);
  const int nb = max(b_hi - b_lo, 0);
  constexpr int W_TMA = 4, W_MMA = 5;

  if (warp == W_TMA && lane == 0) {
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmQ);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&s_empty[s], 4);
    }
    mbar_init(q_ready, 1);
    fence_mbar_init();
  }
  if (warp == W_MMA) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // the queries / row statistics come from the preceding kernels
  pdl_launch_dependents();
  if (warp < 4) {
    if constexpr (MODE != 1) {
      const int r = warp * 32 + lane;
      const int rr = mt * ST_ROWS + r;
      float m = INFINITY, wgt = 0.f;  // padding rows: exp(s - inf) * 0 = 0
      if (rr < R) {
        const int grow = (rr / G) * a.Hq + hk * G + rr % G;
        if constexpr (MODE == 2) {
          const float2 ms = a.row_ms[grow];
          m = ms.x;
          wgt = ms.y;
        } else {
          m = 0.f;
          wgt = 1.f;
        }
      }
      s_m[r] = m;
      s_w[r] = wgt;
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");  // s_m / s_w read by all four compute warps
  }

  if (warp == W_TMA) {
    if (nb > 0 && elect_one()) {
      // the three bf16 query terms of this (kv head, row tile), split by score_split_kernel
      mbar_arrive_expect_tx(q_ready, ST_SPLITS * C::Q_SPLIT);
      for (int sp = 0; sp < ST_SPLITS; ++sp)
#pragma unroll
        for (int at = 0; at < C::ATOMS; ++at)
          tma_load_2d(sQ + sp * C::Q_SPLIT + at * (ST_ROWS * 128), &tmQ, q_ready, at * 64,
                      (sp * a.Hkv + hk) * r_pad + mt * ST_ROWS);
      for (int i = 0; i < nb; ++i) {
        const int st = i % C::STAGES;
        mbar_wait(&k_empty[st], ((i / C::STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&k_full[st], C::K_BYTES);
        const int key0 = a.key_row0 + (b_lo + i) * ST_KEYS;
#pragma unroll
        for (int at = 0; at < C::ATOMS; ++at)
          tma_load_2d(sK + st * C::K_BYTES + at * (ST_KEYS * 128), &tmK, &k_full[st], hk * DH + at * 64, key0);
      }
    }
  } else if (warp == W_MMA) {
    if (nb > 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(128, 128, 0, 0);
      const uint64_t dq = umma_desc_sw128(smem_u32(sQ), 16, 1024);
      const uint64_t dk = umma_desc_sw128(smem_u32(sK), 16, 1024);
      mbar_wait(q_ready, 0);
      for (int i = 0; i < nb; ++i) {
        const int st = i % C::STAGES, tb = i & 1;
        mbar_wait(&k_full[st], (i / C::STAGES) & 1);
        mbar_wait(&s_empty[tb], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t k0 = dk + ((st * C::K_BYTES) >> 4);
          const uint32_t d = tmem + tb * 128;
#pragma unroll
          for (int sp = 0; sp < ST_SPLITS; ++sp) {
            const uint64_t q0 = dq + ((sp * C::Q_SPLIT) >> 4);
#pragma unroll
            for (int kk = 0; kk < DH / 16; ++kk) {
              const uint32_t off = ((kk >> 2) * (128 * 128) + (kk & 3) * 32) >> 4;
              // pass 1: D[rows][keys] = Q K^T; pass 2: D[keys][rows] = K Q^T
              if constexpr (MODE == 1)
                umma_bf16_ss(d, q0 + off, k0 + off, idesc, (sp | kk) != 0);
              else
                umma_bf16_ss(d, k0 + off, q0 + off, idesc, (sp | kk) != 0);
            }
          }
          umma_commit(&s_full[tb]);
          umma_commit(&k_empty[st]);
        }
        __syncwarp();
      }
    }
  } else {
    // ---- compute warps: one thread per TMEM lane
    const int ln = warp * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
    float m_run = -INFINITY, l_run = 0.f;  // pass 1 (row ln)
    for (int i = 0; i < nb; ++i) {
      const int st = i & 1;
      const int key0 = (b_lo + i) * ST_KEYS;
      mbar_wait(&s_full[st], (i >> 1) & 1);
      tc_fence_after();
      uint32_t s[128];
#pragma unroll
      for (int cc = 0; cc < 4; ++cc)
        tmem_ld32(lane_base + st * 128 + cc * 32, *reinterpret_cast<uint32_t(*)[32]>(&s[cc * 32]));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[st]);  // TMEM buffer free for block i + 2
      if constexpr (MODE == 1) {
        // columns = keys key0 + c; natural-log units x = s * scale
        const int nvalid = min(ST_KEYS, a.n_keys - key0);
        if (nvalid < ST_KEYS) {
#pragma unroll
          for (int c = 0; c < 128; ++c)
            if (c >= nvalid) s[c] = 0xff800000u;  // -inf: past the chunk keys
        }
        // four independent chains (ILP), combined in a fixed order
        float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < 128; ++c) mx4[c & 3] = fmaxf(mx4[c & 3], __uint_as_float(s[c]));
        const float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * a.scale;
        const float m_new = fmaxf(m_run, mx);
        const float mb = m_new * LOG2E, cs = a.scale * LOG2E;
        float z4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int c = 0; c < 128; ++c) z4[c & 3] += ex2_approx(__fmaf_rn(__uint_as_float(s[c]), cs, -mb));
        const float z = (z4[0] + z4[1]) + (z4[2] + z4[3]);
        l_run = (m_run == -INFINITY ? 0.f : l_run * ex2_approx((m_run - m_new) * LOG2E)) + z;
        m_run = m_new;
      } else {
        // columns = query rows r of this tile; lane = key key0 + ln
        float acc4[4] = {0.f, 0.f, 0.f, 0.f};
        const float cs = a.scale * LOG2E;
#pragma unroll
        for (int c = 0; c < 128; ++c) {
          if constexpr (MODE == 2)
            acc4[c & 3] = __fmaf_rn(ex2_approx(__fmaf_rn(__uint_as_float(s[c]), cs, -s_m[c] * LOG2E)), s_w[c],
                                    acc4[c & 3]);
          else
            acc4[c & 3] = __fmaf_rn(__uint_as_float(s[c]) * a.scale, s_w[c], acc4[c & 3]);
        }
        const float acc = (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);
        if (key0 + ln < a.n_keys)
          a.col_part[((size_t)hk * gridDim.y + mt) * a.n_keys + key0 + ln] = acc;
      }
    }
    if constexpr (MODE == 1) {
      const int rr = mt * ST_ROWS + ln;
      if (rr < R) {
        const int grow = (rr / G) * a.Hq + hk * G + rr % G;
        a.part_ms[(size_t)grp * nrows_tot + grow] = make_float2(m_run, l_run);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == W_MMA) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

// Exact three-term bf16 split of the fp32 final-layer queries into the tiles
// the scoring passes TMA-load: qs[(sp * Hkv + hk) * r_pad + rr][dh] with
// row rr = t * G + g of kv head hk (zero rows pad each head to r_pad).
__global__ void score_split_kernel(const float* __restrict__ q, int nq, int Hq, int Hkv, int dh, int r_pad,
                                   bf16* __restrict__ qs) {
  pdl_wait();
  pdl_launch_dependents();
  const int G = Hq / Hkv, R = nq * G, c8 = dh / 8;
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long)Hkv * r_pad * c8) return;
  const int c = (int)(idx % c8);
  const int rr = (int)((idx / c8) % r_pad);
  const int hk = (int)(idx / ((long)c8 * r_pad));
  float x[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (rr < R) {
    const float4* src = reinterpret_cast<const float4*>(q + ((size_t)(rr / G) * Hq + hk * G + rr % G) * dh + c * 8);
    const float4 a = src[0], b = src[1];
    x[0] = a.x, x[1] = a.y, x[2] = a.z, x[3] = a.w, x[4] = b.x, x[5] = b.y, x[6] = b.z, x[7] = b.w;
  }
  uint32_t w[ST_SPLITS][4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint32_t h0 = bf16_bits(x[2 * e]), h1 = bf16_bits(x[2 * e + 1]);
    const float r0 = x[2 * e] - bf16_val(h0), r1 = x[2 * e + 1] - bf16_val(h1);  // exact
    const uint32_t m0 = bf16_bits(r0), m1 = bf16_bits(r1);
    const uint32_t l0 = bf16_bits(r0 - bf16_val(m0)), l1 = bf16_bits(r1 - bf16_val(m1));
    w[0][e] = h0 | (h1 << 16);
    w[1][e] = m0 | (m1 << 16);
    w[2][e] = l0 | (l1 << 16);
  }
#pragma unroll
  for (int sp = 0; sp < ST_SPLITS; ++sp)
    *reinterpret_cast<uint4*>(qs + ((size_t)(sp * Hkv + hk) * r_pad + rr) * dh + c * 8) =
        make_uint4(w[sp][0], w[sp][1], w[sp][2], w[sp][3]);
}

// scores[j] = sum over the Hkv x row-tile partials in a fixed order
__global__ void score_head_sum_kernel(const float* __restrict__ col_part, int n_part, int n_keys,
                                      float* __restrict__ scores) {
  pdl_wait();
  pdl_launch_dependents();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_keys) return;
  float s = 0.f;
  for (int p = 0; p < n_part; ++p) s += col_part[(size_t)p * n_keys + j];
  scores[j] = s;
}

template <int DH>
int score_tc_dh(const ScoreArgs& a, cudaStream_t stream) {
  using C = ScoreCfg<DH>;
  CUtensorMap tk;
  // final-layer fused K [rows][Hkv*dh]; rows past the chunk range are zero-filled
  if (!make_tmap_2d(&tk, a.k, (uint64_t)a.key_row0 + a.n_keys, (uint64_t)a.Hkv * DH, (uint64_t)a.Hkv * DH, ST_KEYS))
    return -1;
  const int G = a.Hq / a.Hkv;
  const int n_mt = (a.nq * G + ST_ROWS - 1) / ST_ROWS;
  const int r_pad = n_mt * ST_ROWS;
  CUtensorMap tq;
  if (!make_tmap_2d(&tq, a.q_split, (uint64_t)ST_SPLITS * a.Hkv * r_pad, DH, DH, ST_ROWS)) return -1;
  const int n_blocks = (a.n_keys + ST_KEYS - 1) / ST_KEYS;
  // at most one wave of CTAs (one per SM: the tile uses ~160 KB of shared
  // memory); each walks a contiguous group of key blocks
  const int per_group = a.Hkv * n_mt;
  const int max_groups = std::max(1, num_sms() / per_group);
  int bpg = (n_blocks + max_groups - 1) / max_groups;
  if (bpg < 1) bpg = 1;
  const int n_groups = (n_blocks + bpg - 1) / bpg;
  const dim3 grid(n_groups, n_mt, a.Hkv);
  const int smem = (int)C::SMEM;
  int launches = 1;
  {
    const long n = (long)a.Hkv * r_pad * (DH / 8);
    launch_pdl(score_split_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, stream, a.q, a.nq, a.Hq, a.Hkv,
               DH, r_pad, a.q_split);
  }
  if (!a.raw) {
    smem_attr_once(score_tc_kernel<1, DH>, smem);
    smem_attr_once(score_tc_kernel<2, DH>, smem);
    launch_pdl(score_tc_kernel<1, DH>, grid, dim3(ST_THREADS), smem, stream, tk, tq, a, bpg, r_pad);
    launches += 1 + score_combine(a, n_groups, stream);
    launch_pdl(score_tc_kernel<2, DH>, grid, dim3(ST_THREADS), smem, stream, tk, tq, a, bpg, r_pad);
  } else {
    smem_attr_once(score_tc_kernel<3, DH>, smem);
    launch_pdl(score_tc_kernel<3, DH>, grid, dim3(ST_THREADS), smem, stream, tk, tq, a, bpg, r_pad);
  }
  launch_pdl(score_head_sum_kernel, dim3((a.n_keys + 255) / 256), dim3(256), 0, stream,
             (const float*)a.col_part, (int)(a.Hkv * n_mt), a.n_keys, a.scores);
  launches += 2;
  return cudaPeekAtLastError() == cudaSuccess ? launches : -1;
}

}  // namespace

size_t score_col_part_elems(int nq, int Hq, int Hkv, int n_keys) {
  const int G = Hq / Hkv;
  return (size_t)Hkv * ((nq * G + ST_ROWS - 1) / ST_ROWS) * n_keys;
}
size_t score_q_split_elems(int nq, int Hq, int Hkv, int dh) {
  const int G = Hq / Hkv;
  return (size_t)ST_SPLITS * Hkv * ((nq * G + ST_ROWS - 1) / ST_ROWS) * ST_ROWS * dh;
}

int qg_score_tc(const ScoreArgs& a, cudaStream_t stream) {
  if (a.n_keys <= 0) return 0;
  if (a.Hq % a.Hkv != 0 || !a.col_part || !a.q_split) return -1;
  if (a.dh == 128) return score_tc_dh<128>(a, stream);
  if (a.dh == 64) return score_tc_dh<64>(a, stream);
  return -1;
}

}  // namespace fragk
