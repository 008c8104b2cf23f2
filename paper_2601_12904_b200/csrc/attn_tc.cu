// K6 on the 5th-gen tensor cores: sparse-Q causal attention over the fused KV
// cache.
//
// Only the selected query rows (critical + question, ascending fused rows p_i)
// are computed; row i attends fused rows [0, p_i]. The fused cache already
// holds this layer's fresh K/V at every selected row (scattered by the QKV
// GEMM epilogue), so stale entries are replaced and earlier critical tokens'
// fresh K/V are visible in the same pass.
//
// One CTA = two 128-row query tiles (each 128/G tokens x G heads of one GQA
// group; both share every K/V tile) x one key split. 10 warps:
//   warp 0      TMA: both Q tiles once; K and V tiles (64 keys x dh, SW128)
//               into a 2-stage ring.
//   warp 1      TMEM alloc (512 cols) + single-thread tcgen05.mma issue, per
//               K/V tile j:  S_A(j), S_B(j)   = Q_t K_j^T   (M=128, N=64, K=dh)
//                            O_A += P_A(j-1) V_{j-1},  O_B += P_B(j-1) V_{j-1}
//               S is double-buffered per tile so S(j+1) overlaps softmax(j).
//   warps 2-5   softmax of tile A, warps 6-9 softmax of tile B: one thread per
//               query row (TMEM lane) -> two softmax warps per SM sub-partition.
//               Online softmax in log2 units with lazy O rescale (> 2^8), P ->
//               bf16 -> swizzled smem (K-major UMMA A operand); V is the
//               MN-major B operand straight from its TMA tile.
// Split-KV partials (O normalised per split + LSE) are merged by
// attn_combine_kernel (attn.cu).
#include <cuda.h>

#include <cfloat>

#include "kernels.h"
#include "ptx.cuh"

namespace fragk {

namespace {

constexpr int AT_ROWS = 128;  // rows per query tile
constexpr int AT_QT = 2;      // query tiles per CTA
constexpr int AT_KEYS = 64;   // keys per K/V tile
constexpr int AT_THREADS = 320;
constexpr int KV_STAGES = 3;  // K/V ring depth (2 tiles of prefetch)
constexpr float RESCALE_THRESH = 8.0f;  // log2 units

template <int DH>
struct AttCfg {
  static constexpr int ATOMS = DH / 64;                         // 64-column swizzle atoms per row
  static constexpr uint32_t Q_TILE = AT_ROWS * DH * 2;          // [ATOMS][128][64]
  static constexpr uint32_t KV_ATOM = AT_KEYS * 128;            // [64 keys][64 cols] bf16
  static constexpr uint32_t KV_BYTES = AT_KEYS * DH * 2;        // K (or V) per stage
  static constexpr uint32_t P_BYTES = AT_ROWS * AT_KEYS * 2;    // [128][64] one atom
  static constexpr size_t SMEM =
      1024 + AT_QT * (size_t)Q_TILE + 2 * KV_STAGES * (size_t)KV_BYTES + AT_QT * 2 * (size_t)P_BYTES + 512;
  // TMEM columns per query tile: S0, S1 (64 each), O (DH)
  static constexpr uint32_t T_S0 = 0, T_S1 = 64, T_O = 128, T_TILE = 256;
};

template <int DH>
__global__ void __launch_bounds__(AT_THREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const AttnArgs a, int G, int n_qblocks) {
  using C = AttCfg<DH>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                          // [QT][Q_TILE]
  uint8_t* sK = sQ + AT_QT * C::Q_TILE;        // [2 stages][KV_BYTES]
  uint8_t* sV = sK + KV_STAGES * C::KV_BYTES;  // [stages][KV_BYTES]
  uint8_t* sP = sV + KV_STAGES * C::KV_BYTES;  // [QT][2 buffers][P_BYTES]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sP + AT_QT * 2 * C::P_BYTES);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;      // [KV_STAGES]
  uint64_t* v_full = bar + 4;      // [KV_STAGES]
  uint64_t* pv_done = bar + 7;     // [KV_STAGES]: PV_A(j), PV_B(j) of the tile in that stage complete
  uint64_t* s_full = bar + 10;     // [QT][2]
  uint64_t* s_empty = bar + 14;    // [QT][2]
  uint64_t* p_full = bar + 18;     // [QT][2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 22);

  const int warp = warp_id(), lane = lane_id();
  const int qb = n_qblocks - 1 - (int)blockIdx.x;  // heaviest (latest rows) first
  const int hk = blockIdx.y;
  const int split = blockIdx.z;
  const int tok_per_tile = AT_ROWS / G;
  const int t0 = qb * AT_QT * tok_per_tile;
  const int t_end = min(t0 + AT_QT * tok_per_tile, a.M);
  const int n_qt = (t_end - t0 + tok_per_tile - 1) / tok_per_tile;  // live query tiles (1 or 2)
  const int p_max = a.rows[t_end - 1];
  const int k_lo = a.n_splits > 1 ? split * a.split_keys : 0;
  int k_hi = p_max + 1;
  if (a.n_splits > 1) k_hi = min(k_hi, (split + 1) * a.split_keys);
  const int n_tiles = k_hi > k_lo ? (k_hi - k_lo + AT_KEYS - 1) / AT_KEYS : 0;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < KV_STAGES; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&pv_done[s], 1);
    }
    for (int i = 0; i < AT_QT * 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 4);
      mbar_init(&p_full[i], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (n_tiles > 0 && elect_one()) {
      mbar_arrive_expect_tx(q_full, n_qt * C::Q_TILE);
      for (int t = 0; t < n_qt; ++t)
#pragma unroll
        for (int at = 0; at < C::ATOMS; ++at)
          tma_load_3d(sQ + t * C::Q_TILE + at * (AT_ROWS * 128), &tmQ, q_full, at * 64, hk * G,
                      t0 + t * tok_per_tile);
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j % KV_STAGES;
        const int use = j / KV_STAGES;
        mbar_wait(&pv_done[st], (use & 1) ^ 1);  // stage free once PV(j - KV_STAGES) is done
        const int key0 = k_lo + j * AT_KEYS;
        mbar_arrive_expect_tx(&k_full[st], C::KV_BYTES);
#pragma unroll
        for (int at = 0; at < C::ATOMS; ++at)
          tma_load_2d(sK + st * C::KV_BYTES + at * C::KV_ATOM, &tmK, &k_full[st], hk * DH + at * 64, key0);
        mbar_arrive_expect_tx(&v_full[st], C::KV_BYTES);
#pragma unroll
        for (int at = 0; at < C::ATOMS; ++at)
          tma_load_2d(sV + st * C::KV_BYTES + at * C::KV_ATOM, &tmV, &v_full[st], hk * DH + at * 64, key0);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (n_tiles > 0) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(AT_ROWS, AT_KEYS, 0, 0);
      constexpr uint32_t idesc_o = umma_idesc_bf16(AT_ROWS, DH, 0, 1);
      mbar_wait(q_full, 0);
      tc_fence_after();
      auto issue_pv = [&](int j) {
        const int st = j % KV_STAGES, pb = j & 1;
        mbar_wait(&v_full[st], (j / KV_STAGES) & 1);
        for (int t = 0; t < n_qt; ++t) {
          mbar_wait(&p_full[t * 2 + pb], (j >> 1) & 1);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t p_base = smem_u32(sP + (t * 2 + pb) * C::P_BYTES);
            const uint32_t v_base = smem_u32(sV + st * C::KV_BYTES);
#pragma unroll
            for (int kk = 0; kk < AT_KEYS / 16; ++kk) {
              const uint64_t ad = umma_desc_sw128(p_base + kk * 32, 16, 1024);
              // V tile [64 keys][64-dh atoms], MN-major: K step = 16 key rows = 2048 B,
              // next 64-wide dh atom at LBO = 64 keys * 128 B.
              const uint64_t bd = umma_desc_sw128(v_base + kk * 2048, C::KV_ATOM, 1024);
              umma_bf16_ss(tmem + t * C::T_TILE + C::T_O, ad, bd, idesc_o, (j | kk) != 0);
            }
            // one commit per PV pair: it frees the K/V stage and P buffers (j%2)
            // and publishes O for the softmax rescale / epilogue
            if (t == n_qt - 1) umma_commit(&pv_done[st]);
          }
          __syncwarp();
        }
      };
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j % KV_STAGES, sb = j & 1;
        mbar_wait(&k_full[st], (j / KV_STAGES) & 1);
        for (int t = 0; t < n_qt; ++t) {
          if (j >= 2) mbar_wait(&s_empty[t * 2 + sb], ((j >> 1) - 1) & 1);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t q_base = smem_u32(sQ + t * C::Q_TILE);
            const uint32_t k_base = smem_u32(sK + st * C::KV_BYTES);
#pragma unroll
            for (int kk = 0; kk < DH / 16; ++kk) {
              const uint64_t ad = umma_desc_sw128(q_base + (kk >> 2) * (AT_ROWS * 128) + (kk & 3) * 32, 16, 1024);
              const uint64_t bd = umma_desc_sw128(k_base + (kk >> 2) * C::KV_ATOM + (kk & 3) * 32, 16, 1024);
              umma_bf16_ss(tmem + t * C::T_TILE + (sb ? C::T_S1 : C::T_S0), ad, bd, idesc_s, kk != 0);
            }
            umma_commit(&s_full[t * 2 + sb]);
          }
          __syncwarp();
        }
        if (j >= 1) issue_pv(j - 1);
      }
      issue_pv(n_tiles - 1);
    }
  } else {
    // ------------------------------------------------------------ softmax / epilogue
    const int t = (warp - 2) >> 2;  // query tile of this warp group
    if (t < n_qt) {
      const int q4 = warp & 3;
      const int r = q4 * 32 + lane;  // query row within the tile = TMEM lane
      const int tl = (t * AT_ROWS + r) / G;
      const int tok = t0 + tl;
      const int head = hk * G + r % G;
      const bool live = tok < a.M;
      const int prow = live ? a.rows[tok] : -1;
      const int p_min = a.rows[t0 + t * tok_per_tile];
      const uint32_t lane_base = tmem + ((uint32_t)(q4 * 32) << 16) + t * C::T_TILE;
      const float c = a.scale * 1.4426950408889634f;
      uint64_t* sf = s_full + t * 2;
      uint64_t* se = s_empty + t * 2;
      uint64_t* pf = p_full + t * 2;
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j & 1;
        const int key0 = k_lo + j * AT_KEYS;
        mbar_wait(&sf[st], (j >> 1) & 1);
        tc_fence_after();
        uint32_t s[AT_KEYS];
        tmem_ld32(lane_base + (st ? C::T_S1 : C::T_S0), *reinterpret_cast<uint32_t(*)[32]>(&s[0]));
        tmem_ld32(lane_base + (st ? C::T_S1 : C::T_S0) + 32, *reinterpret_cast<uint32_t(*)[32]>(&s[32]));
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&se[st]);
        // causal mask by position (keys > p_row or beyond the split), raw scores
        const int lim = min(prow, k_hi - 1) - key0;
        if ((key0 + AT_KEYS - 1 > p_min) || (key0 + AT_KEYS > k_hi)) {
#pragma unroll
          for (int k = 0; k < AT_KEYS; ++k)
            if (k > lim) s[k] = 0xff800000u;  // -inf
        }
        float mx8[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) mx8[e] = __uint_as_float(s[e]);
#pragma unroll
        for (int k = 8; k < AT_KEYS; k += 8)
#pragma unroll
          for (int e = 0; e < 8; ++e) mx8[e] = fmaxf(mx8[e], __uint_as_float(s[k + e]));
        const float mt = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                               fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * c;
        // lazy rescale: only when the max grows by more than 2^8
        const bool grow = mt > m_used + RESCALE_THRESH || (m_used == -INFINITY && mt != -INFINITY);
        const float m_new = grow ? fmaxf(mt, m_used) : m_used;
        const float alpha = (grow && m_used != -INFINITY) ? ex2_approx(m_used - m_new) : 1.f;
        if (__any_sync(0xffffffffu, grow && m_used != -INFINITY) && j > 0) {
          // rescale this lane quarter's O rows in TMEM; PV(j-1) must have landed
          mbar_wait(&pv_done[(j - 1) % KV_STAGES], ((j - 1) / KV_STAGES) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int cc = 0; cc < DH / 32; ++cc) {
            uint32_t o[32];
            tmem_ld32(lane_base + C::T_O + cc * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            tmem_st32(lane_base + C::T_O + cc * 32, o);
          }
          tmem_st_wait();
        }
        l *= alpha;
        m_used = m_new;
        // P buffer j%2 was last read by PV(j-2): wait for it explicitly (do not rely
        // on commit ordering between different accumulators)
        if (j >= 2) mbar_wait(&pv_done[(j - 2) % KV_STAGES], ((j - 2) / KV_STAGES) & 1);
        // p = 2^(s*c - m): one FFMA + MUFU.EX2 per element; masked s = -inf -> 0
        const float mneg = m_used == -INFINITY ? 0.f : -m_used;
        uint8_t* prow_smem = sP + (t * 2 + st) * C::P_BYTES + r * 128;
        float rs8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int ch = 0; ch < AT_KEYS / 8; ++ch) {
          float p[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            p[e] = ex2_approx(__fmaf_rn(__uint_as_float(s[ch * 8 + e]), c, mneg));
            rs8[e] += p[e];
          }
          uint4 pk;
          pk.x = pack_bf16(p[0], p[1]);
          pk.y = pack_bf16(p[2], p[3]);
          pk.z = pack_bf16(p[4], p[5]);
          pk.w = pack_bf16(p[6], p[7]);
          *reinterpret_cast<uint4*>(prow_smem + ((ch ^ (r & 7)) << 4)) = pk;
        }
        l += ((rs8[0] + rs8[1]) + (rs8[2] + rs8[3])) + ((rs8[4] + rs8[5]) + (rs8[6] + rs8[7]));
        fence_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&pf[st]);
      }
      // ---- epilogue
      if (n_tiles > 0) {
        mbar_wait(&pv_done[(n_tiles - 1) % KV_STAGES], ((n_tiles - 1) / KV_STAGES) & 1);
        tc_fence_after();
      }
      const float inv = l > 0.f ? 1.f / l : 0.f;
      const size_t qi = (size_t)tok * a.Hq + head;
#pragma unroll 1
      for (int cc = 0; cc < DH / 32; ++cc) {
        uint32_t o[32];
        if (n_tiles > 0) {
          tmem_ld32(lane_base + C::T_O + cc * 32, o);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = 0u;
        }
        if (!live) continue;
        if (a.n_splits > 1) {
          float4* po = reinterpret_cast<float4*>(a.part_o + ((size_t)split * a.M * a.Hq + qi) * DH + cc * 32);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            po[e] = make_float4(__uint_as_float(o[4 * e]) * inv, __uint_as_float(o[4 * e + 1]) * inv,
                                __uint_as_float(o[4 * e + 2]) * inv, __uint_as_float(o[4 * e + 3]) * inv);
        } else {
          uint4* po = reinterpret_cast<uint4*>(a.out + qi * DH + cc * 32);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            uint4 v;
            v.x = pack_bf16(__uint_as_float(o[8 * e + 0]) * inv, __uint_as_float(o[8 * e + 1]) * inv);
            v.y = pack_bf16(__uint_as_float(o[8 * e + 2]) * inv, __uint_as_float(o[8 * e + 3]) * inv);
            v.z = pack_bf16(__uint_as_float(o[8 * e + 4]) * inv, __uint_as_float(o[8 * e + 5]) * inv);
            v.w = pack_bf16(__uint_as_float(o[8 * e + 6]) * inv, __uint_as_float(o[8 * e + 7]) * inv);
            po[e] = v;
          }
        }
      }
      if (live && a.n_splits > 1) {
        // natural-log LSE of the scaled scores: m (log2 units) * ln2 + ln(l)
        a.part_lse[(size_t)split * a.M * a.Hq + qi] =
            l > 0.f ? m_used * 0.6931471805599453f + __logf(l) : -INFINITY;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace

int attn_rows_per_cta() { return AT_ROWS * AT_QT; }

int attn_tc_launch(const AttnArgs& a, int G, int n_qblocks, cudaStream_t stream) {
  CUtensorMap tq, tk, tv;
  // Q [M][Hq][dh] viewed as (dh, Hq, M); box (64, G, 128/G)
  if (!make_tmap_3d(&tq, a.q, a.dh, a.Hq, a.M, a.dh, (uint64_t)a.Hq * a.dh, 64, G, AT_ROWS / G)) return -1;
  // K/V layer [T][Hkv*dh]; box (64, 64 keys)
  if (!make_tmap_2d(&tk, a.k, a.T, (uint64_t)a.Hkv * a.dh, (uint64_t)a.Hkv * a.dh, AT_KEYS)) return -1;
  if (!make_tmap_2d(&tv, a.v, a.T, (uint64_t)a.Hkv * a.dh, (uint64_t)a.Hkv * a.dh, AT_KEYS)) return -1;
  dim3 grid(n_qblocks, a.Hkv, a.n_splits);
  if (a.dh == 128) {
    smem_attr_once(attn_tc_kernel<128>, (int)AttCfg<128>::SMEM);
    attn_tc_kernel<128><<<grid, AT_THREADS, AttCfg<128>::SMEM, stream>>>(tq, tk, tv, a, G, n_qblocks);
  } else if (a.dh == 64) {
    smem_attr_once(attn_tc_kernel<64>, (int)AttCfg<64>::SMEM);
    attn_tc_kernel<64><<<grid, AT_THREADS, AttCfg<64>::SMEM, stream>>>(tq, tk, tv, a, G, n_qblocks);
  } else {
    return -1;
  }
  return 1;
}

}  // namespace fragk
