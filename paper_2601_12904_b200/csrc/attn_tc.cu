// K6 on the 5th-gen tensor cores: sparse-Q causal attention over the fused KV
// cache.
//
// Only the selected query rows (critical + question, ascending fused rows p_i)
// are computed; row i attends fused rows [0, p_i]. The fused cache already
// holds this layer's fresh K/V at every selected row (scattered by the QKV
// GEMM epilogue), so stale entries are replaced and earlier critical tokens'
// fresh K/V are visible in the same pass.
//
// One CTA = two 128-row query tiles A, B (each 128/G tokens x G heads of one
// GQA group; both share every K/V tile) x one key split. 10 warps:
//   warp 8      TMA: both Q tiles once; K and V tiles (128 keys x dh, SW128)
//               into a 2-stage ring.
//   warp 9      TMEM alloc (512 cols) + single-thread tcgen05.mma issue in a
//               ping-pong order so one tile's softmax overlaps the other
//               tile's MMAs:
//                 S_A(0) S_B(0) | PV_A(0) S_A(1) | PV_B(0) S_B(1) | PV_A(1) ...
//               S_t = Q_t K^T (M=128, N=128 keys, K=dh, both operands from smem)
//               O_t += P_t V  (M=128, N=dh, K=128 keys, P from TMEM, V MN-major smem)
//   warps 0-3   softmax of tile A, warps 4-7 of tile B: one thread per query
//               row (TMEM lane). tcgen05.ld S, causal mask by position, online
//               softmax in log2 units (lazy O rescale when the max grows > 2^8),
//               P packed bf16 and tcgen05.st back over the S columns.
// TMEM per tile: [S | P aliased](128 cols) + O (128 cols); the in-order tensor
// pipe orders PV_t(j)'s read of P before S_t(j+1) overwrites those columns.
// Split-KV partials (O normalised per split + LSE) are merged by
// attn_combine_kernel (attn.cu).
#include <cuda.h>

#include <cfloat>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels.h"
#include "ptx.cuh"

namespace fragk {

namespace {

constexpr int AT_ROWS = 128;  // rows per query tile
constexpr int AT_QT = 2;      // query tiles per CTA
constexpr int AT_KEYS = 128;  // keys per K/V tile
constexpr int AT_THREADS = 320;
constexpr float RESCALE_THRESH = 8.0f;  // log2 units
constexpr int kDefaultPoly = 0;
constexpr int kQtmPoly = 4;  // Q-in-TMEM kernel: every 4th exp pair on the FMA pipe  // measured: MUFU-only is fastest at dh=128 (tools/attn_bench.py)

template <int DH>
struct AttCfg {
  static constexpr int ATOMS = DH / 64;                    // 64-column swizzle atoms per row
  static constexpr uint32_t Q_TILE = AT_ROWS * DH * 2;     // [ATOMS][128][64]
  static constexpr uint32_t KV_ATOM = AT_KEYS * 128;       // [128 keys][64 cols] bf16
  static constexpr uint32_t KV_BYTES = AT_KEYS * DH * 2;   // K (or V) per stage
  static constexpr size_t SMEM = 1024 + AT_QT * (size_t)Q_TILE + 4 * (size_t)KV_BYTES + 256;
  // DUAL (one query tile): the second Q slot holds a third K/V stage
  static constexpr size_t SMEM_DUAL = 1024 + (size_t)Q_TILE + 6 * (size_t)KV_BYTES + 256;
  static_assert(SMEM_DUAL <= 232448, "3-stage attention tile exceeds the 227 KB shared-memory limit");
  static constexpr uint32_t T_S = 0, T_O = 128, T_TILE = 256;  // TMEM columns per tile
  static_assert(SMEM <= 232448, "attention tile exceeds the 227 KB shared-memory limit");
};

// ---------------------------------------------------------------- shared V pages
// VSH kernels read V in place from the store's records (AttnArgs::vsegs): the
// TMA warp loads each 128-key V tile from its primary segment's tensor map
// (rows outside that record arrive as zeros: OOB fill), and one more warp, the
// patch warp, writes the rows the box cannot supply -- rows of other segments
// and this request's fresh rows (critical rows from the per-request plan,
// question / decoded rows by rule) from the exclusive region -- into the
// swizzled tile, then releases it to the MMA warp (v_ready). The tile the MMA
// consumes is byte-identical to the private fused-cache tile.
template <int DH, int NS>
__device__ __forceinline__ void vpatch_loop(const AttnArgs& a, int hk, int k_lo, int k_hi, int n_tiles, uint8_t* sV,
                                            uint64_t* v_full, uint64_t* v_ready, int lane) {
  // Each patched row is one TMA box (64 cols x 1 row) per 64-column atom,
  // written straight into its swizzled place in the tile (the 128-byte
  // swizzle follows the shared-memory address) and counted on v_ready: no
  // registers, no proxy fence, and the warp moves on to the next tile while
  // the rows are in flight. The next tile's plan entries are loaded ahead.
  constexpr int ATOMS = DH / 64;
  constexpr uint32_t KV_ATOM = AT_KEYS * 128;
  constexpr uint32_t KV_BYTES = AT_KEYS * DH * 2;
  const int tile0 = k_lo / AT_KEYS;
  const int* starts = a.vtile;
  int e_lo = __ldg(starts + tile0), e_mid = __ldg(starts + tile0 + 1);
  int e_hi = n_tiles > 1 ? __ldg(starts + tile0 + 2) : e_mid;
  unsigned long long ent[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) ent[q] = lane + 32 * q < e_mid - e_lo ? __ldg(a.vent + e_lo + lane + 32 * q) : 0ull;
  for (int j = 0; j < n_tiles; ++j) {
    const int st = j % NS;
    const int key0 = k_lo + j * AT_KEYS;
    const int tr0 = max(key0, a.tail_row0), tr1 = min(key0 + AT_KEYS, k_hi);
    const int n_ent = e_mid - e_lo;
    const int n = n_ent + max(0, tr1 - tr0);  // <= 128: planned rows < tail_row0 <= tail rows
    // next tile's entries (in flight across the wait below)
    unsigned long long nxt[4];
    int e_after = e_hi;
    if (j + 1 < n_tiles) {
#pragma unroll
      for (int q = 0; q < 4; ++q) nxt[q] = lane + 32 * q < e_hi - e_mid ? __ldg(a.vent + e_mid + lane + 32 * q) : 0ull;
      if (j + 2 < n_tiles) e_after = __ldg(starts + tile0 + j + 3);
    }
    uint8_t* sv = sV + st * KV_BYTES;
    mbar_wait(&v_full[st], (j / NS) & 1);  // the primary box has landed: patch over it
    if (a.trace && blockIdx.x == 0 && lane == 0 && j < 256)  // tooling: primary landed | patch rows << 48
      a.trace[1024 + j * 4 + 3] = ((unsigned long long)clock64() & 0xffffffffffffull) | ((unsigned long long)n << 48);
    if (lane == 0) mbar_arrive_expect_tx(&v_ready[st], (uint32_t)n * DH * 2);
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int p = lane + 32 * q;
      if (p < n) {
        const CUtensorMap* tm;
        int y, r;
        if (p < n_ent) {
          const unsigned long long e = ent[q];
          r = (int)(e & 127);
          const int seg = (int)((e >> 8) & 0xffffff);
          y = (int)(e >> 32);
          tm = seg == 0 ? a.vx_map : &a.vsegs[seg - 1].tmap1;
        } else {
          const int row = tr0 + (p - n_ent);
          r = row - key0;
          y = a.tail_slot0 + row - a.tail_row0;
          tm = a.vx_map;
        }
#pragma unroll
        for (int at = 0; at < ATOMS; ++at)
          tma_load_3d(sv + at * KV_ATOM + r * 128, tm, &v_ready[st], hk * DH + at * 64, y, a.layer);
      }
    }
    if (j + 1 < n_tiles) {
#pragma unroll
      for (int q = 0; q < 4; ++q) ent[q] = nxt[q];
    }
    e_lo = e_mid;
    e_mid = e_hi;
    e_hi = e_after;
  }
}

// POLY: every POLY-th pair of P elements takes the FMA-pipe 2^x (ex2_poly)
// instead of MUFU.EX2, balancing the two pipes (0 = all MUFU).
// DUAL (one query tile per CTA: the question pass and decode): the two tile
// slots share the single Q tile and split every 128-key tile in halves
// (slot t takes keys t*64 .. t*64+63), so both softmax warp groups and the
// MMA ping-pong stay busy; the two partial softmaxes (m, l, O) are merged in
// the epilogue.
// SPLIT (default for dh=128): two softmax threads per query
// row (16 softmax warps: warps w and w+4 of a tile share TMEM lanes and take
// 64 of the 128 keys each, the row max exchanged through shared memory).
template <int DH, int POLY, bool DUAL = false, bool SPLIT = false, bool VSH = false>
__global__ void __launch_bounds__(SPLIT ? 576 : (VSH ? AT_THREADS + 32 : AT_THREADS), 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const AttnArgs a, int G, int n_qblocks) {
  using C = AttCfg<DH>;
  static_assert(!(DUAL && SPLIT), "DUAL and SPLIT are separate variants");
  static_assert(!VSH || DUAL, "shared V pages: the DUAL (one query tile) variant");
  constexpr int KT = DUAL ? AT_KEYS / 2 : AT_KEYS;  // keys per tile slot per K/V tile
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // K/V ring depth: 2 stages next to two Q tiles; DUAL keeps one Q tile and
  // spends the other slot on a third stage (the question pass / decode CTAs
  // stream ~8 K/V tiles each and are latency-bound on the ring)
  constexpr int NS = DUAL ? 3 : 2;
  uint8_t* sQ = smem;                                    // [QT or 1][Q_TILE]
  uint8_t* sK = sQ + (DUAL ? 1 : AT_QT) * C::Q_TILE;     // [NS stages][KV_BYTES]
  uint8_t* sV = sK + NS * C::KV_BYTES;                   // [NS stages][KV_BYTES]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sV + NS * C::KV_BYTES);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;              // [NS]
  uint64_t* v_full = bar + 1 + NS;         // [NS]
  uint64_t* kv_empty = bar + 1 + 2 * NS;   // [NS]
  uint64_t* s_full = bar + 1 + 3 * NS;     // [QT]
  uint64_t* p_full = s_full + AT_QT;       // [QT]
  uint64_t* pv_done = p_full + AT_QT;      // [QT]
  uint64_t* v_ready = pv_done + AT_QT;     // [NS] VSH: V tile patched
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(v_ready + NS);

  const int warp = warp_id(), lane = lane_id();
  // global longest-first order: q-block work grows with its row positions, so
  // dispatch (q-block desc) x (kv head) makes the hardware's greedy CTA
  // scheduler an LPT schedule across all heads (the tail wave is the lightest)
  const int qb = n_qblocks - 1 - (int)blockIdx.x / a.Hkv;
  const int hk = (int)blockIdx.x % a.Hkv;
  const int split = blockIdx.z;
  const int tok_per_tile = AT_ROWS / G;
  const int t0 = qb * AT_QT * tok_per_tile;
  const int t_end = min(t0 + AT_QT * tok_per_tile, a.M);
  const int n_qt = (t_end - t0 + tok_per_tile - 1) / tok_per_tile;  // live query tiles (1 or 2)
  const int k_lo = a.n_splits > 1 ? split * a.split_keys : 0;

  // warps 0-3 softmax A, 4-7 softmax B, 8 TMA, 9 MMA (the highest warp id wins
  // issue arbitration on its sub-partition, which keeps MMA issue off the
  // softmax critical path)
  constexpr int W_TMA = SPLIT ? 16 : 8, W_MMA = W_TMA + 1, W_PATCH = W_TMA + 2;
  if constexpr (VSH)
    if (warp == W_TMA)
      for (int i = lane; i < a.n_vseg; i += 32) {
        tma_prefetch_desc(&a.vsegs[i].tmap);
        tma_prefetch_desc(&a.vsegs[i].tmap1);
      }
  if (warp == W_TMA && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    if constexpr (!VSH) tma_prefetch_desc(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&kv_empty[s], 1);
      mbar_init(&v_ready[s], 1);
    }
    for (int t = 0; t < AT_QT; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], SPLIT ? 8 : 4);
      mbar_init(&pv_done[t], 1);
    }
    fence_mbar_init();
  }
  if (warp == W_MMA) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // PDL: the prologue above overlapped the producing kernel's tail; the plan
  // rows, Q and the fused K/V rows are read only after this point
  pdl_wait();
  pdl_launch_dependents();
  const int p_max = a.rows[t_end - 1] - a.row_base;
  int k_hi = p_max + 1;
  if (a.n_splits > 1) k_hi = min(k_hi, (split + 1) * a.split_keys);
  const int n_tiles = k_hi > k_lo ? (k_hi - k_lo + AT_KEYS - 1) / AT_KEYS : 0;
  const int n_slots = DUAL ? AT_QT : n_qt;  // tile slots in use (DUAL: both on the one Q tile)

  if (warp == W_TMA) {
    // ------------------------------------------------------------ TMA producer
    if (n_tiles > 0 && elect_one()) {
      mbar_arrive_expect_tx(q_full, n_qt * C::Q_TILE);
      for (int t = 0; t < n_qt; ++t)
#pragma unroll
        for (int at = 0; at < C::ATOMS; ++at)
          tma_load_3d(sQ + t * C::Q_TILE + at * (AT_ROWS * 128), &tmQ, q_full, at * 64, hk * G,
                      t0 + t * tok_per_tile);
      const int tile0 = k_lo / AT_KEYS;
      int2 pr = make_int2(0, 0);  // VSH: this tile's primary V segment + row coordinate
      if constexpr (VSH) pr = __ldg(a.vprim + tile0);
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j % NS;
        int2 pr_next = pr;
        if constexpr (VSH)
          if (j + 1 < n_tiles) pr_next = __ldg(a.vprim + tile0 + j + 1);  // in flight across the wait
        mbar_wait(&kv_empty[st], ((j / NS) & 1) ^ 1);  // PV(j-NS) done with this stage
        const int key0 = k_lo + j * AT_KEYS;
        mbar_arrive_expect_tx(&k_full[st], C::KV_BYTES);
#pragma unroll
        for (int at = 0; at < C::ATOMS; ++at)
          tma_load_2d(sK + st * C::KV_BYTES + at * C::KV_ATOM, &tmK, &k_full[st], hk * DH + at * 64, key0);
        mbar_arrive_expect_tx(&v_full[st], C::KV_BYTES);
        if constexpr (VSH) {
          const CUtensorMap* tm = &a.vsegs[pr.x].tmap;
#pragma unroll
          for (int at = 0; at < C::ATOMS; ++at)
            tma_load_3d(sV + st * C::KV_BYTES + at * C::KV_ATOM, tm, &v_full[st], hk * DH + at * 64, pr.y, a.layer);
        } else {
#pragma unroll
          for (int at = 0; at < C::ATOMS; ++at)
            tma_load_2d(sV + st * C::KV_BYTES + at * C::KV_ATOM, &tmV, &v_full[st], hk * DH + at * 64, key0);
        }
        pr = pr_next;
      }
      // consume the last NS kv_empty phases (no phase completes unobserved)
      for (int j = n_tiles > NS ? n_tiles - NS : 0; j < n_tiles; ++j) mbar_wait(&kv_empty[j % NS], (j / NS) & 1);
    }
  } else if (warp == W_MMA) {
    // ------------------------------------------------------------ MMA issuer
    if (n_tiles > 0) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(AT_ROWS, KT, 0, 0);
      constexpr uint32_t idesc_o = umma_idesc_bf16(AT_ROWS, DH, 0, 1);
      mbar_wait(q_full, 0);
      // descriptor templates: only the 14-bit start-address field changes per MMA
      const uint64_t dq = umma_desc_sw128(smem_u32(sQ), 16, 1024);
      const uint64_t dk = umma_desc_sw128(smem_u32(sK), 16, 1024);
      const uint64_t dv = umma_desc_sw128(smem_u32(sV), C::KV_ATOM, 1024);
      auto issue_s = [&](int t, int j) {
        const int st = j % NS;
        mbar_wait(&k_full[st], (j / NS) & 1);
        tc_fence_after();
        if (a.trace && blockIdx.x == 0 && lane == 0 && j < 256) a.trace[(t * 256 + j) * 4 + 2] = clock64();
        if (elect_one()) {
          const uint64_t q0 = dq + (((DUAL ? 0 : t) * C::Q_TILE) >> 4);
          // DUAL: keys t*64.. of the tile = 8 KB into each 128-key K atom
          const uint64_t k0 = dk + ((st * C::KV_BYTES + (DUAL ? t * KT * 128 : 0)) >> 4);
          const uint32_t d_tmem = tmem + t * C::T_TILE + C::T_S;
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk) {
            const uint32_t off = ((kk >> 2) * (AT_ROWS * 128) + (kk & 3) * 32) >> 4;  // Q/K atoms are 128 rows
            umma_bf16_ss(d_tmem, q0 + off, k0 + off, idesc_s, kk != 0);
          }
          umma_commit(&s_full[t]);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int t, int j) {
        const int st = j % NS;
        mbar_wait(&p_full[t], j & 1);
        tc_fence_after();
        if (a.trace && blockIdx.x == 0 && lane == 0 && j < 256) a.trace[(t * 256 + j) * 4 + 3] = clock64();
        if (elect_one()) {
          const uint64_t v0 = dv + ((st * C::KV_BYTES) >> 4);
          const uint32_t d_tmem = tmem + t * C::T_TILE + C::T_O;
          const uint32_t p_tmem = tmem + t * C::T_TILE + C::T_S;
#pragma unroll
          for (int kk = 0; kk < KT / 16; ++kk) {
            // P: 16 keys = 8 packed bf16x2 TMEM columns; V: 16 key rows = 2048 B,
            // MN-major, next 64-wide dh atom at LBO = 128 keys * 128 B
            const int vrow = (DUAL ? t * KT : 0) + kk * 16;
            umma_bf16_ts(d_tmem, p_tmem + kk * 8, v0 + ((vrow * 128) >> 4), idesc_o, (j | kk) != 0);
          }
          umma_commit(&pv_done[t]);
          if (t == n_slots - 1) umma_commit(&kv_empty[st]);
        }
        __syncwarp();
      };
      for (int t = 0; t < n_slots; ++t) issue_s(t, 0);
      for (int j = 0; j < n_tiles; ++j) {
        mbar_wait(&v_full[j % NS], (j / NS) & 1);
        if constexpr (VSH) mbar_wait(&v_ready[j % NS], (j / NS) & 1);
        for (int t = 0; t < n_slots; ++t) {
          issue_pv(t, j);
          if (j + 1 < n_tiles) issue_s(t, j + 1);
        }
      }
    }
  } else if (VSH && warp == W_PATCH) {
    // ------------------------------------------------------------ V patch warp (shared V pages)
    if (n_tiles > 0) vpatch_loop<DH, NS>(a, hk, k_lo, k_hi, n_tiles, sV, v_full, v_ready, lane);
  } else if constexpr (SPLIT) {
    // ------------------------------------------------------------ split-row softmax / epilogue
    __shared__ float xm[AT_QT][2][2][AT_ROWS];  // [tile][iteration parity][half][row] partial max
    __shared__ float xl[AT_QT][2][AT_ROWS];     // [tile][half][row] partial row sum
    const int t = warp >> 3, half = (warp >> 2) & 1, q4 = warp & 3;
    if (t < n_qt) {
      const int r = q4 * 32 + lane;
      const int tl = (t * AT_ROWS + r) / G;
      const int tok = t0 + tl;
      const int head = hk * G + r % G;
      const bool live = tok < a.M;
      const int prow = live ? a.rows[tok] - a.row_base : -1;
      const int p_min = a.rows[t0 + t * tok_per_tile] - a.row_base;
      const uint32_t lane_base = tmem + ((uint32_t)(q4 * 32) << 16) + t * C::T_TILE;
      const float c = a.scale * 1.4426950408889634f;
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < n_tiles; ++j) {
        const int key0 = k_lo + j * AT_KEYS + half * 64;
        mbar_wait(&s_full[t], j & 1);
        // S(j) was committed after PV(j-1): consume every pv_done phase (free)
        if (j > 0) mbar_wait(&pv_done[t], (j - 1) & 1);
        tc_fence_after();
        uint32_t sa[32], sb[32];
        tmem_ld32(lane_base + C::T_S + half * 64, sa);
        tmem_ld32(lane_base + C::T_S + half * 64 + 32, sb);
        tmem_ld_wait();
#define SV(k) (*((k) < 32 ? &sa[(k) & 31] : &sb[(k) & 31]))
        const int lim = min(prow, k_hi - 1) - key0;
        if ((key0 + 63 > p_min) || (key0 + 64 > k_hi)) {
#pragma unroll
          for (int k = 0; k < 64; ++k)
            if (k > lim) SV(k) = 0xff800000u;
        }
        float mx4[4] = {__uint_as_float(sa[0]), __uint_as_float(sa[1]), __uint_as_float(sa[2]), __uint_as_float(sa[3])};
#pragma unroll
        for (int k = 4; k < 60; k += 8)
#pragma unroll
          for (int e = 0; e < 4; ++e) mx4[e] = fmax3(mx4[e], __uint_as_float(SV(k + e)), __uint_as_float(SV(k + 4 + e)));
#pragma unroll
        for (int e = 0; e < 4; ++e) mx4[e] = fmaxf(mx4[e], __uint_as_float(sb[28 + e]));
        xm[t][j & 1][half][r] = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
        asm volatile("bar.sync %0, 256;" ::"r"(1 + t) : "memory");
        const float mt = fmaxf(xm[t][j & 1][0][r], xm[t][j & 1][1][r]) * c;
        const bool grow = mt > m_used + RESCALE_THRESH || (m_used == -INFINITY && mt != -INFINITY);
        const float m_new = grow ? fmaxf(mt, m_used) : m_used;
        const float alpha = (grow && m_used != -INFINITY) ? ex2_approx(m_used - m_new) : 1.f;
        const bool resc = grow && m_used != -INFINITY;
        l *= alpha;
        m_used = m_new;
        const float mneg = m_used == -INFINITY ? 0.f : -m_used;
        float rs8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int e = 0; e < 32; ++e) {  // packed in place: sa[e] <- P(keys 2e, 2e+1)
          const float p0 = ex2_approx(__fmaf_rn(__uint_as_float(SV(2 * e)), c, mneg));
          const float p1 = ex2_approx(__fmaf_rn(__uint_as_float(SV(2 * e + 1)), c, mneg));
          rs8[(2 * e) & 7] += p0;
          rs8[(2 * e + 1) & 7] += p1;
          sa[e] = pack_bf16(p0, p1);
        }
#undef SV
        tmem_st32(lane_base + C::T_S + half * 32, sa);  // P of keys half*64.. = packed columns half*32..
        l += ((rs8[0] + rs8[1]) + (rs8[2] + rs8[3])) + ((rs8[4] + rs8[5]) + (rs8[6] + rs8[7]));
        tmem_st_wait();
        // O rescale after P is out (fewer live registers); PV(j) waits on p_full anyway
        if (__any_sync(0xffffffffu, resc) && j > 0) {
#pragma unroll 1
          for (int cc = 0; cc < DH / 64; ++cc) {  // this half's 64 of the DH O columns
            uint32_t o[32];
            const uint32_t ocol = C::T_O + half * (DH / 2) + cc * 32;
            tmem_ld32(lane_base + ocol, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            tmem_st32(lane_base + ocol, o);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[t]);
        if (a.trace && blockIdx.x == 0 && lane == 0 && q4 == 0 && half == 0 && j < 256) {
          a.trace[(t * 256 + j) * 4 + 0] = 0;  // (S-ready stamp not taken in this variant)
          a.trace[(t * 256 + j) * 4 + 1] = clock64();
        }
      }
      // ---- epilogue: row sum = both halves' partial sums (same reference max)
      if (n_tiles > 0) {
        mbar_wait(&pv_done[t], (n_tiles - 1) & 1);
        tc_fence_after();
      }
      xl[t][half][r] = l;
      asm volatile("bar.sync %0, 256;" ::"r"(1 + t) : "memory");
      const float lt = xl[t][0][r] + xl[t][1][r];
      const float inv = lt > 0.f ? 1.f / lt : 0.f;
      const size_t qi = (size_t)tok * a.Hq + head;
#pragma unroll 1
      for (int cc = 0; cc < DH / 64; ++cc) {
        uint32_t o[32];
        const int dcol = half * (DH / 2) + cc * 32;
        if (n_tiles > 0) {
          tmem_ld32(lane_base + C::T_O + dcol, o);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = 0u;
        }
        if (!live) continue;
        if (a.n_splits > 1) {
          float4* po = reinterpret_cast<float4*>(a.part_o + ((size_t)split * a.M * a.Hq + qi) * DH + dcol);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            po[e] = make_float4(__uint_as_float(o[4 * e]) * inv, __uint_as_float(o[4 * e + 1]) * inv,
                                __uint_as_float(o[4 * e + 2]) * inv, __uint_as_float(o[4 * e + 3]) * inv);
        } else {
          uint4* po = reinterpret_cast<uint4*>(a.out + qi * DH + dcol);
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
      if (live && half == 0 && a.n_splits > 1)
        a.part_lse[(size_t)split * a.M * a.Hq + qi] =
            lt > 0.f ? m_used * 0.6931471805599453f + __logf(lt) : -INFINITY;
    }
  } else {
    // ------------------------------------------------------------ softmax / epilogue
    const int t = warp >> 2;  // query tile (DUAL: key half) of this warp group
    const int tq = DUAL ? 0 : t;  // query tile of this warp group's rows
    if (t < n_slots) {
      const int q4 = warp & 3;
      const int r = q4 * 32 + lane;  // query row within the tile = TMEM lane
      const int tl = (tq * AT_ROWS + r) / G;
      const int tok = t0 + tl;
      const int head = hk * G + r % G;
      const bool live = tok < a.M;
      const int prow = live ? a.rows[tok] - a.row_base : -1;
      const int p_min = a.rows[t0 + tq * tok_per_tile] - a.row_base;
      const uint32_t lane_base = tmem + ((uint32_t)(q4 * 32) << 16) + t * C::T_TILE;
      const float c = a.scale * 1.4426950408889634f;
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < n_tiles; ++j) {
        const int key0 = k_lo + j * AT_KEYS + (DUAL ? t * KT : 0);
        mbar_wait(&s_full[t], j & 1);
        // S(j) was committed after PV(j-1): consume every pv_done phase (free)
        if (j > 0) mbar_wait(&pv_done[t], (j - 1) & 1);
        tc_fence_after();
        if (a.trace && blockIdx.x == 0 && lane == 0 && (warp & 3) == 0 && j < 256)
          a.trace[(t * 256 + j) * 4 + 0] = clock64();
        uint32_t s[KT];
#pragma unroll
        for (int cc = 0; cc < KT / 32; ++cc)
          tmem_ld32(lane_base + C::T_S + cc * 32, *reinterpret_cast<uint32_t(*)[32]>(&s[cc * 32]));
        tmem_ld_wait();
        // causal mask by position (keys > p_row or beyond the split), raw scores
        const int lim = min(prow, k_hi - 1) - key0;
        if ((key0 + KT - 1 > p_min) || (key0 + KT > k_hi)) {
#pragma unroll
          for (int k = 0; k < KT; ++k)
            if (k > lim) s[k] = 0xff800000u;  // -inf
        }
        float mx8[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) mx8[e] = __uint_as_float(s[e]);
#pragma unroll
        for (int k = 8; k < KT - 8; k += 16)
#pragma unroll
          for (int e = 0; e < 8; ++e) mx8[e] = fmax3(mx8[e], __uint_as_float(s[k + e]), __uint_as_float(s[k + 8 + e]));
#pragma unroll
        for (int e = 0; e < 8; ++e) mx8[e] = fmaxf(mx8[e], __uint_as_float(s[KT - 8 + e]));
        const float mt = fmax3(fmax3(mx8[0], mx8[1], mx8[2]), fmax3(mx8[3], mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])) * c;
        // lazy rescale: only when the max grows by more than 2^8
        const bool grow = mt > m_used + RESCALE_THRESH || (m_used == -INFINITY && mt != -INFINITY);
        const float m_new = grow ? fmaxf(mt, m_used) : m_used;
        const float alpha = (grow && m_used != -INFINITY) ? ex2_approx(m_used - m_new) : 1.f;
        if (__any_sync(0xffffffffu, grow && m_used != -INFINITY) && j > 0) {
          // rescale this lane quarter's O rows in TMEM; PV_t(j-1) has landed (waited above)
#pragma unroll 1
          for (int cc = 0; cc < DH / 32; ++cc) {
            uint32_t o[32];
            tmem_ld32(lane_base + C::T_O + cc * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            tmem_st32(lane_base + C::T_O + cc * 32, o);
          }
        }
        l *= alpha;
        m_used = m_new;
        // p = 2^(s*c - m): one FFMA + MUFU.EX2 per element; masked s = -inf -> 0.
        // P (bf16 pairs) overwrites the first 64 S columns of this tile.
        const float mneg = m_used == -INFINITY ? 0.f : -m_used;
        float rs8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int half = 0; half < KT / 64; ++half) {
          uint32_t pk[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const int k = half * 64 + 2 * e;
            const float x0 = __fmaf_rn(__uint_as_float(s[k]), c, mneg);
            const float x1 = __fmaf_rn(__uint_as_float(s[k + 1]), c, mneg);
            const bool poly = POLY > 0 && (e % (POLY > 0 ? POLY : 1)) == POLY - 1;
            const float p0 = poly ? ex2_poly(x0) : ex2_approx(x0);
            const float p1 = poly ? ex2_poly(x1) : ex2_approx(x1);
            rs8[(2 * e) & 7] += p0;
            rs8[(2 * e + 1) & 7] += p1;
            pk[e] = pack_bf16(p0, p1);
          }
          tmem_st32(lane_base + C::T_S + half * 32, pk);
        }
        l += ((rs8[0] + rs8[1]) + (rs8[2] + rs8[3])) + ((rs8[4] + rs8[5]) + (rs8[6] + rs8[7]));
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[t]);
        if (a.trace && blockIdx.x == 0 && lane == 0 && (warp & 3) == 0 && j < 256)
          a.trace[(t * 256 + j) * 4 + 1] = clock64();
      }
      // ---- epilogue
      if (n_tiles > 0) {
        mbar_wait(&pv_done[t], (n_tiles - 1) & 1);
        tc_fence_after();
      }
      float a0 = 1.f, a1 = 0.f;  // DUAL: weights of the two key halves' partial O
      if constexpr (DUAL) {
        // slot 1 publishes (m, l) of its key half in the unused second Q slot;
        // slot 0 merges: m = max, O = (O0 2^(m0-m) + O1 2^(m1-m)) / (l0 2^(m0-m) + l1 2^(m1-m))
        float* pub = reinterpret_cast<float*>(sQ + C::Q_TILE);
        if (t == 1) {
          pub[r] = m_used;
          pub[AT_ROWS + r] = l;
        }
        asm volatile("bar.sync 2, 256;" ::: "memory");
        if (t == 1) {
          m_used = -INFINITY;  // nothing to store for slot 1
          l = 0.f;
        } else {
          const float m1 = pub[r], l1 = pub[AT_ROWS + r];
          if (n_tiles > 0) {
            mbar_wait(&pv_done[1], (n_tiles - 1) & 1);
            tc_fence_after();
          }
          const float m = fmaxf(m_used, m1);
          a0 = m_used == -INFINITY ? 0.f : ex2_approx(m_used - m);
          a1 = m1 == -INFINITY ? 0.f : ex2_approx(m1 - m);
          l = l * a0 + l1 * a1;
          m_used = m;
        }
      }
      const float inv = l > 0.f ? 1.f / l : 0.f;
      const size_t qi = (size_t)tok * a.Hq + head;
      const bool writer = !(DUAL && t == 1);  // warp-uniform: slot 1's half was merged by slot 0
#pragma unroll 1
      for (int cc = 0; cc < (writer ? DH / 32 : 0); ++cc) {
        uint32_t o[32];
        if (n_tiles > 0) {
          tmem_ld32(lane_base + C::T_O + cc * 32, o);
          if constexpr (DUAL) {
            uint32_t o1[32];
            tmem_ld32(lane_base + C::T_TILE + C::T_O + cc * 32, o1);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e)
              o[e] = __float_as_uint(__uint_as_float(o[e]) * a0 + __uint_as_float(o1[e]) * a1);
          } else {
            tmem_ld_wait();
          }
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
      if (writer && live && a.n_splits > 1) {
        // natural-log LSE of the scaled scores: m (log2 units) * ln2 + ln(l)
        a.part_lse[(size_t)split * a.M * a.Hq + qi] =
            l > 0.f ? m_used * 0.6931471805599453f + __logf(l) : -INFINITY;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == W_MMA) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ---------------------------------------------------------------- Q in TMEM
// One 128-row query tile per CTA (128/G tokens x G heads of one GQA group)
// with Q resident in TMEM as the A operand of S = Q K^T (tcgen05.mma with A
// from TMEM): the S MMA reads only K from shared memory. The r01 kernels
// read Q and K from shared memory (8 KB per K=16 step = the whole 128 B/clk
// port), which bound them at ~1370 cycles per tile pair against 1024 ideal,
// and their per-tile chain softmax -> PV -> next S serialised each tile.
// TMEM (448 of 512 cols): S/P double buffer 2 x 128 (P aliased into the
// first 64 cols of its S buffer) + O (DH) + Q (DH/2 packed bf16). With two S
// buffers the tensor pipe computes S(u+1) -- and PV(u-1) -- while the
// softmax works on S(u):
//   S(0) S(1) | PV(0) S(2) | PV(1) S(3) | ...
// 16 softmax warps: warp w owns TMEM lane quarter w%4 (its SMSP) and key
// columns 32*(w/4).. of each 128-key slice; the row max is exchanged through
// shared memory behind one named barrier per lane quarter and slice (the same
// barrier orders every warp's S load before any P store over those columns).
// An O rescale (lazy, > 2^8) waits for PV(u-1); otherwise the softmax of
// slice u never waits on the tensor pipe.
template <int DH, int PE>
__global__ void __launch_bounds__(576, 1)
    attn_qtm_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                    const AttnArgs a, int G, int n_qblocks) {
  constexpr int ATOMS = DH / 64;
  constexpr uint32_t KV_ATOM = AT_KEYS * 128;
  constexpr uint32_t KV_BYTES = AT_KEYS * DH * 2;
  // separate K and V rings: a K stage is free once S(u) is done, a V stage
  // once PV(u) is; the V ring is the deeper one (a V tile is consumed a tile
  // later than its K, and with shared V pages it also waits for its patches)
  constexpr int NSK = DH == 128 ? 2 : 4, NSV = DH == 128 ? 4 : 8;
  // S buffer b at b*128; O; the row sums L (16 cols, every one = sum_k P); Q
  constexpr uint32_t T_S0 = 0, T_O = 256, T_L = T_O + DH, T_Q = 448;
  constexpr int QC = DH / 8;                           // packed Q columns per column-group warp
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;                    // [NSK][KV_BYTES]
  uint8_t* sV = sK + NSK * KV_BYTES;     // [NSV][KV_BYTES]
  uint8_t* sOnes = sV + NSV * KV_BYTES;  // 2 KB of bf16 1.0: B operand of the row-sum MMA (N=16)
  uint64_t* bar = reinterpret_cast<uint64_t*>(sOnes + 2048);
  uint64_t* k_full = bar;                // [NSK]
  uint64_t* k_empty = k_full + NSK;      // [NSK]
  uint64_t* v_full = k_empty + NSK;      // [NSV]
  uint64_t* v_empty = v_full + NSV;      // [NSV]
  uint64_t* q_full = v_empty + NSV;
  uint64_t* s_full = q_full + 1;        // [2] per S buffer
  uint64_t* p_full = s_full + 2;        // [2]
  uint64_t* pv_done = p_full + 2;
  // every PV (and row-sum) MMA complete: the epilogue cannot use pv_done, whose
  // last two phases may both be outstanding when the softmax finishes its last
  // tile (a parity wait cannot tell phase n-1 from n-3)
  uint64_t* o_done = pv_done + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 1);
  __shared__ float xm[2][4][AT_ROWS];   // [slice parity][column group][row] partial max

  const int warp = warp_id(), lane = lane_id();
  const int qb = n_qblocks - 1 - (int)blockIdx.x / a.Hkv;  // longest-first (see attn_tc_kernel)
  const int hk = (int)blockIdx.x % a.Hkv;
  const int split = blockIdx.z;
  const int tok_per_tile = AT_ROWS / G;
  const int t0 = qb * tok_per_tile;
  const int t_end = min(t0 + tok_per_tile, a.M);
  const int k_lo = a.n_splits > 1 ? split * a.split_keys : 0;
  constexpr int W_TMA = 16, W_MMA = 17;
  if (warp == W_TMA && lane == 0) {
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    for (int s = 0; s < NSK; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < NSV; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    mbar_init(q_full, 16);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], 16);
    }
    mbar_init(pv_done, 1);
    mbar_init(o_done, 1);
    fence_mbar_init();
  }
  if (warp == W_MMA) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();
  const int p_max = a.rows[t_end - 1] - a.row_base;
  int k_hi = p_max + 1;
  if (a.n_splits > 1) k_hi = min(k_hi, (split + 1) * a.split_keys);
  const int n_tiles = k_hi > k_lo ? (k_hi - k_lo + AT_KEYS - 1) / AT_KEYS : 0;

  if (warp == W_TMA) {
    if (n_tiles > 0 && elect_one()) {
      for (int j = 0; j < n_tiles; ++j) {
        const int sv = j % NSV, sk = j % NSK;
        const int key0 = k_lo + j * AT_KEYS;
        // V(j) first: the V ring runs further ahead (its stage frees at PV(j-NSV),
        // long before K(j)'s at S(j-NSK))
        mbar_wait(&v_empty[sv], ((j / NSV) & 1) ^ 1);
        mbar_arrive_expect_tx(&v_full[sv], KV_BYTES);
#pragma unroll
        for (int at = 0; at < ATOMS; ++at)
          tma_load_2d(sV + sv * KV_BYTES + at * KV_ATOM, &tmV, &v_full[sv], hk * DH + at * 64, key0);
        mbar_wait(&k_empty[sk], ((j / NSK) & 1) ^ 1);
        mbar_arrive_expect_tx(&k_full[sk], KV_BYTES);
#pragma unroll
        for (int at = 0; at < ATOMS; ++at)
          tma_load_2d(sK + sk * KV_BYTES + at * KV_ATOM, &tmK, &k_full[sk], hk * DH + at * 64, key0);
      }
      // consume the last phases of both rings (no phase completes unobserved)
      for (int j = n_tiles > NSV ? n_tiles - NSV : 0; j < n_tiles; ++j) mbar_wait(&v_empty[j % NSV], (j / NSV) & 1);
      for (int j = n_tiles > NSK ? n_tiles - NSK : 0; j < n_tiles; ++j) mbar_wait(&k_empty[j % NSK], (j / NSK) & 1);
    }
  } else if (warp == W_MMA) {
    if (n_tiles > 0) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(AT_ROWS, AT_KEYS, 0, 0);
      constexpr uint32_t idesc_o = umma_idesc_bf16(AT_ROWS, DH, 0, 1);
      constexpr uint32_t idesc_l = umma_idesc_bf16(AT_ROWS, 16, 0, 0);
      const uint64_t d_ones = umma_desc_sw128(smem_u32(sOnes), 16, 1024);
      const uint64_t dk = umma_desc_sw128(smem_u32(sK), 16, 1024);
      const uint64_t dv = umma_desc_sw128(smem_u32(sV), KV_ATOM, 1024);
      mbar_wait(q_full, 0);
      tc_fence_after();
      auto issue_s = [&](int u) {
        const int st = u % NSK;
        mbar_wait(&k_full[st], (u / NSK) & 1);
        tc_fence_after();
        if (a.trace && blockIdx.x == 0 && lane == 0 && u < 256) a.trace[u * 4 + 2] = clock64();
        if (elect_one()) {
          const uint64_t k0 = dk + ((st * KV_BYTES) >> 4);
          const uint32_t d_tmem = tmem + T_S0 + (u & 1) * 128;
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk) {
            const uint32_t off = ((kk >> 2) * KV_ATOM + (kk & 3) * 32) >> 4;
            umma_bf16_ts(d_tmem, tmem + T_Q + kk * 8, k0 + off, idesc_s, kk != 0);
          }
          umma_commit(&s_full[u & 1]);
          umma_commit(&k_empty[st]);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int u) {
        const int st = u % NSV;
        // V(u) landed and PV(u-1) done are independent of slice u's softmax:
        // observe them first, so that P(u) is the only wait between the last
        // softmax warp's arrival and the PV issue (the tensor pipe idles there)
        mbar_wait(&v_full[st], (u / NSV) & 1);
        // observe pv_done phase u-1 (no phase completes unwaited; PV(u-2) is
        // known complete here -- S(u) was, and the pipe is in order -- so the
        // parity is unambiguous); PV(u-1) has normally finished while the
        // softmax of slice u ran
        if (u > 0) mbar_wait(pv_done, (u - 1) & 1);
        mbar_wait(&p_full[u & 1], (u >> 1) & 1);
        tc_fence_after();
        if (a.trace && blockIdx.x == 0 && lane == 0 && u < 256) a.trace[u * 4 + 3] = clock64();
        if (elect_one()) {
          const uint64_t v0 = dv + ((st * KV_BYTES) >> 4);
          const uint32_t p_tmem = tmem + T_S0 + (u & 1) * 128;
#pragma unroll
          for (int kk = 0; kk < AT_KEYS / 16; ++kk)
            umma_bf16_ts(tmem + T_O, p_tmem + kk * 8, v0 + ((kk * 16 * 128) >> 4), idesc_o, (u | kk) != 0);
          // row sums on the tensor pipe: L += P . 1 (the bf16 P that also multiplies V)
#pragma unroll
          for (int kk = 0; kk < AT_KEYS / 16; ++kk)
            umma_bf16_ts(tmem + T_L, p_tmem + kk * 8, d_ones, idesc_l, (u | kk) != 0);
          umma_commit(pv_done);
          umma_commit(&v_empty[st]);
        }
        __syncwarp();
      };
      issue_s(0);
      if (n_tiles > 1) issue_s(1);
      for (int u = 0; u < n_tiles; ++u) {
        issue_pv(u);
        if (u + 2 < n_tiles) issue_s(u + 2);
      }
      if (elect_one()) umma_commit(o_done);
      __syncwarp();
      mbar_wait(pv_done, (n_tiles - 1) & 1);  // the last phase (PV(n-2) observed above)
    }
  } else {
    // ------------------------------------------------------------ softmax / epilogue (16 warps)
    const int q4 = warp & 3, cg = warp >> 2;
    const int r = q4 * 32 + lane;
    const int tok = t0 + r / G;
    const int head = hk * G + r % G;
    const bool live = tok < a.M;
    const int prow = live ? a.rows[tok] - a.row_base : -1;
    const int p_min = a.rows[t0] - a.row_base;
    const uint32_t lane_base = tmem + ((uint32_t)(q4 * 32) << 16);
    const size_t qi = (size_t)tok * a.Hq + head;
    const int nbar = 1 + q4;  // named barrier of this lane quarter (its 4 column-group warps)
    {  // Q row, this warp's DH/4 columns -> TMEM (A operand of S)
      uint32_t qr[QC];
      if (live) {
        const uint4* src = reinterpret_cast<const uint4*>(a.q + qi * DH + cg * (DH / 4));
#pragma unroll
        for (int e = 0; e < QC / 4; ++e) {
          const uint4 v = __ldg(src + e);
          qr[4 * e] = v.x, qr[4 * e + 1] = v.y, qr[4 * e + 2] = v.z, qr[4 * e + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int e = 0; e < QC; ++e) qr[e] = 0u;
      }
      if constexpr (QC == 16)
        tmem_st16(lane_base + T_Q + cg * QC, qr);
      else
        tmem_st8(lane_base + T_Q + cg * QC, qr);
      if (cg == 0 && r < 64) {  // 32 bytes each of the 2 KB ones tile (16 rows x 128 B, SW128)
        uint4* o1 = reinterpret_cast<uint4*>(sOnes) + 2 * r;
        const uint4 one = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
        o1[0] = one;
        o1[1] = one;
        fence_async_smem();  // generic writes -> visible to the tensor pipe's reads
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(q_full);
    }
    const float c = a.scale * 1.4426950408889634f;
    float m_used = -INFINITY;
    for (int u = 0; u < n_tiles; ++u) {
      const int b = u & 1;
      const int key0 = k_lo + u * AT_KEYS + cg * 32;
      mbar_wait(&s_full[b], (u >> 1) & 1);
      tc_fence_after();
      if (a.trace && blockIdx.x == 0 && lane == 0 && warp == 0 && u < 256) a.trace[u * 4 + 0] = clock64();
      uint32_t s[32];
      tmem_ld32(lane_base + T_S0 + b * 128 + cg * 32, s);
      tmem_ld_wait();
      if (a.trace && blockIdx.x == 0 && lane == 0 && warp == 0 && u < 256) a.trace[1024 + u * 4 + 0] = clock64();
      const int lim = min(prow, k_hi - 1) - key0;
      if ((key0 + 31 > p_min) || (key0 + 32 > k_hi)) {
#pragma unroll
        for (int k = 0; k < 32; ++k)
          if (k > lim) s[k] = 0xff800000u;
      }
      float mx4[4] = {__uint_as_float(s[0]), __uint_as_float(s[1]), __uint_as_float(s[2]), __uint_as_float(s[3])};
#pragma unroll
      for (int k = 4; k < 28; k += 8)
#pragma unroll
        for (int e = 0; e < 4; ++e) mx4[e] = fmax3(mx4[e], __uint_as_float(s[k + e]), __uint_as_float(s[k + 4 + e]));
#pragma unroll
      for (int e = 0; e < 4; ++e) mx4[e] = fmaxf(mx4[e], __uint_as_float(s[28 + e]));
      const float lmax = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * c;
      // lazy rescale: the row max matters only if some column group's max
      // exceeds m_used + 2^8; one OR-barrier decides for the lane quarter (it
      // also orders every warp's S load before any P store over those columns)
      const bool need = lmax > m_used + RESCALE_THRESH || (m_used == -INFINITY && lmax != -INFINITY);
      float mt = -INFINITY;
      if (bar_red_or(nbar, 128, need)) {
        xm[b][cg][r] = lmax;
        asm volatile("bar.sync %0, 128;" ::"r"(nbar) : "memory");
        mt = fmaxf(fmaxf(xm[b][0][r], xm[b][1][r]), fmaxf(xm[b][2][r], xm[b][3][r]));
      }
      if (a.trace && blockIdx.x == 0 && lane == 0 && warp == 0 && u < 256) a.trace[1024 + u * 4 + 1] = clock64();
      const bool grow = mt > m_used + RESCALE_THRESH || (m_used == -INFINITY && mt != -INFINITY);
      const float m_new = grow ? fmaxf(mt, m_used) : m_used;
      const float alpha = (grow && m_used != -INFINITY) ? ex2_approx(m_used - m_new) : 1.f;
      const bool resc = grow && m_used != -INFINITY;
      m_used = m_new;
      const float mneg = m_used == -INFINITY ? 0.f : -m_used;
      // packed fp32x2 arithmetic (FFMA2 / FADD2: one FMA-pipe issue per two
      // elements); every PE-th pair takes the FMA-pipe polynomial instead of
      // MUFU.EX2: the four softmax warps of an SMSP share its MUFU (4/clk)
      const unsigned long long c2 = f2_pack(c, c), m2 = f2_pack(mneg, mneg);
      uint32_t pk[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const unsigned long long x = f2_fma(f2_pack(__uint_as_float(s[2 * e]), __uint_as_float(s[2 * e + 1])), c2, m2);
        float x0, x1, p0, p1;
        f2_unpack(x, x0, x1);
        if (PE > 0 && (e % (PE > 0 ? PE : 1)) == PE - 1) {
          ex2_poly2(x0, x1, p0, p1);
        } else {
          p0 = ex2_approx(x0);
          p1 = ex2_approx(x1);
        }
        pk[e] = pack_bf16(p0, p1);
      }
      if (a.trace && blockIdx.x == 0 && lane == 0 && warp == 0 && u < 256) a.trace[1024 + u * 4 + 2] = clock64();
      tmem_st16(lane_base + T_S0 + b * 128 + cg * 16, pk);  // P keys cg*32.. = packed cols cg*16..
      if (__any_sync(0xffffffffu, resc) && u > 0) {
        // O holds PV(0..u-1) at the old scale: rescale this warp's DH/4 columns
        // once PV(u-1) has landed; PV(u) waits for p_full below
        mbar_wait(pv_done, (u - 1) & 1);
        tc_fence_after();
        uint32_t o[DH / 4];
        if constexpr (DH / 4 == 32) {
          tmem_ld32(lane_base + T_O + cg * 32, *reinterpret_cast<uint32_t(*)[32]>(o));
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
          tmem_st32(lane_base + T_O + cg * 32, *reinterpret_cast<uint32_t(*)[32]>(o));
        } else {
          uint32_t o32[32];
          tmem_ld32(lane_base + T_O + (cg & 1) * 32, o32);  // DH=64: warps cg<2 own 32 cols each
          tmem_ld_wait();
          if (cg < 2) {
#pragma unroll
            for (int e = 0; e < 32; ++e) o32[e] = __float_as_uint(__uint_as_float(o32[e]) * alpha);
            tmem_st32(lane_base + T_O + cg * 32, o32);
          }
        }
        if (cg == 3) {  // and the row-sum columns
          uint32_t o16[16];
          tmem_ld16(lane_base + T_L, o16);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 16; ++e) o16[e] = __float_as_uint(__uint_as_float(o16[e]) * alpha);
          tmem_st16(lane_base + T_L, o16);
        }
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[b]);
      if (a.trace && blockIdx.x == 0 && lane == 0 && warp == 0 && u < 256) a.trace[u * 4 + 1] = clock64();
      if (a.trace && blockIdx.x == 0 && lane == 0 && u < 256)  // the slice's last softmax warp
        atomicMax(&a.trace[1024 + u * 4 + 3], (unsigned long long)clock64());
    }
    // ---- epilogue: the row sum accumulated by the tensor pipe (T_L)
    float lt = 0.f;
    if (n_tiles > 0) {
      mbar_wait(o_done, 0);
      tc_fence_after();
      uint32_t l16[16];
      tmem_ld16(lane_base + T_L, l16);
      tmem_ld_wait();
      lt = __uint_as_float(l16[0]);
    }
    const float inv = lt > 0.f ? 1.f / lt : 0.f;
    constexpr int OC = DH / 4;  // output columns of this warp
    if (OC == 32 || cg < 2) {
      const int dcol = (OC == 32 ? cg : cg) * 32;
      uint32_t o[32];
      if (n_tiles > 0) {
        tmem_ld32(lane_base + T_O + dcol, o);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] = 0u;
      }
      if (live) {
        if (a.n_splits > 1) {
          float4* po = reinterpret_cast<float4*>(a.part_o + ((size_t)split * a.M * a.Hq + qi) * DH + dcol);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            po[e] = make_float4(__uint_as_float(o[4 * e]) * inv, __uint_as_float(o[4 * e + 1]) * inv,
                                __uint_as_float(o[4 * e + 2]) * inv, __uint_as_float(o[4 * e + 3]) * inv);
        } else {
          uint4* po = reinterpret_cast<uint4*>(a.out + qi * DH + dcol);
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
    } else if (n_tiles > 0) {
      uint32_t o[32];  // DH=64, cg >= 2: keep the warp's tcgen05.ld count uniform (no columns to write)
      tmem_ld32(lane_base + T_O, o);
      tmem_ld_wait();
    }
    if (live && cg == 0 && a.n_splits > 1)
      a.part_lse[(size_t)split * a.M * a.Hq + qi] = lt > 0.f ? m_used * 0.6931471805599453f + __logf(lt) : -INFINITY;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == W_MMA) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int DH>
constexpr size_t qtm_smem() {
  // alignment slack, K + V rings, ones tile, barriers + TMEM slot
  return 1024 + (size_t)(DH == 128 ? 6 : 12) * AT_KEYS * DH * 2 + 2048 + 512;
}
static_assert(qtm_smem<128>() <= 232448 - 4 * 1024 && qtm_smem<64>() <= 232448 - 4 * 1024,
              "Q-in-TMEM attention exceeds 227 KB");

}  // namespace

int attn_rows_per_cta() { return AT_ROWS * AT_QT; }

// The shared-V kernels are the default ones (Q-in-TMEM sparse pass, DUAL
// question pass / decode) with MUFU-only or the default FMA split; the r01
// tuning switches keep the private fused V.
bool attn_shared_v_supported(int dh) {
  if (dh != 64 && dh != 128) return false;
  const char* q = std::getenv("FRAG_ATTN_QTM");
  const char* qq = std::getenv("FRAG_ATTN_QTM_Q");
  const char* p = std::getenv("FRAG_ATTN_POLY");
  const char* qp = std::getenv("FRAG_ATTN_QTM_POLY");
  (void)qq;
  return !(q && q[0] == '0') && !(p && std::atoi(p) != 0) && !(qp && std::atoi(qp) != kQtmPoly);
}

int attn_tc_launch(const AttnArgs& a, int G, int n_qblocks, cudaStream_t stream) {
  CUtensorMap tq, tk, tv;
  // Q [M][Hq][dh] viewed as (dh, Hq, M); box (64, G, 128/G)
  if (!make_tmap_3d(&tq, a.q, a.dh, a.Hq, a.M, a.dh, (uint64_t)a.Hq * a.dh, 64, G, AT_ROWS / G)) return -1;
  // K/V layer [T][Hkv*dh]; box (64, 128 keys)
  if (!make_tmap_2d(&tk, a.k, a.T, (uint64_t)a.Hkv * a.dh, (uint64_t)a.Hkv * a.dh, AT_KEYS)) return -1;
  // shared V pages: V comes from the segments' maps through the patch warp of
  // the one-query-tile (DUAL) kernels; larger passes read a staged V window
  const bool vsh = a.vsegs != nullptr;
  if (vsh && (!attn_shared_v_supported(a.dh) || a.n_vseg < 1 || (a.n_splits > 1 && a.split_keys % AT_KEYS) ||
              a.M > AT_ROWS / G))
    return -1;
  if (vsh)
    tv = tk;  // unused by the VSH kernels
  else if (!make_tmap_2d(&tv, a.v, a.T, (uint64_t)a.Hkv * a.dh, (uint64_t)a.Hkv * a.dh, AT_KEYS))
    return -1;
  dim3 grid(n_qblocks * a.Hkv, 1, a.n_splits);
  // FRAG_ATTN_POLY: tuning knob for the MUFU/FMA exp split (default below)
  static const int poly = [] {
    const char* v = std::getenv("FRAG_ATTN_POLY");
    return v ? std::atoi(v) : kDefaultPoly;
  }();
  // FRAG_ATTN_TRACE=<file>: tooling only (tools/attn_trace.py) -- clock64
  // timeline of CTA 0 (S ready / P done per softmax tile, S / PV issue in the
  // MMA warp) appended to <file> after the launch
  static const char* trace_path = std::getenv("FRAG_ATTN_TRACE");
  static unsigned long long* trace_dev = nullptr;
  AttnArgs at = a;
  if (trace_path) {
    if (!trace_dev) cudaMalloc(&trace_dev, 4 * 256 * 4 * sizeof(unsigned long long));
    cudaMemsetAsync(trace_dev, 0, 4 * 256 * 4 * sizeof(unsigned long long), stream);
    at.trace = trace_dev;
  }
  // two softmax threads per row (default for dh=128; FRAG_ATTN_SPLIT=0 selects
  // the one-thread-per-row kernel): 2-3% faster alone, see DESIGN.md §5
  static const bool split_rows = [] {
    const char* v = std::getenv("FRAG_ATTN_SPLIT");
    return !(v && v[0] == '0');
  }();
  int threads = AT_THREADS;
  auto go = [&](auto kern, int smem) {
    smem_attr_once(kern, smem);
    launch_pdl(kern, grid, dim3(threads), smem, stream, tq, tk, tv, at, G, n_qblocks);
    if (trace_path) {
      unsigned long long h[4 * 256 * 4];
      cudaMemcpyAsync(h, trace_dev, sizeof(h), cudaMemcpyDeviceToHost, stream);
      cudaStreamSynchronize(stream);
      if (FILE* f = std::fopen(trace_path, "ab")) {
        std::fwrite(h, sizeof(h), 1, f);
        std::fclose(f);
      }
    }
  };
  // one query tile per CTA (question pass, decode): split each key tile
  // between the two slots instead of leaving one idle
  // FRAG_ATTN_QTM_Q=1: the one-tile (question pass / decode) case on the Q-in-TMEM kernel too
  static const bool qtm_q = [] {
    const char* v = std::getenv("FRAG_ATTN_QTM_Q");
    return v && v[0] == '1';
  }();
  const bool dual = a.M <= AT_ROWS / G && !qtm_q;
  if (dual && vsh) {
    threads = AT_THREADS + 32;  // + the V patch warp
    if (a.dh == 128)
      go(attn_tc_kernel<128, 0, true, false, true>, (int)AttCfg<128>::SMEM_DUAL);
    else
      go(attn_tc_kernel<64, 0, true, false, true>, (int)AttCfg<64>::SMEM_DUAL);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
  }
  if (dual) {
    if (a.dh == 128)
      go(attn_tc_kernel<128, 0, true>, (int)AttCfg<128>::SMEM_DUAL);
    else if (a.dh == 64)
      go(attn_tc_kernel<64, 0, true>, (int)AttCfg<64>::SMEM_DUAL);
    else
      return -1;
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
  }
  // Q-in-TMEM kernel (default; FRAG_ATTN_QTM=0 selects the r01 SS kernels)
  static const bool qtm = [] {
    const char* v = std::getenv("FRAG_ATTN_QTM");
    return !(v && v[0] == '0');
  }();

  if (qtm && poly == 0 && (a.dh == 128 || a.dh == 64)) {
    const int nqb1 = (a.M + AT_ROWS / G - 1) / (AT_ROWS / G);  // one 128-row tile per CTA
    const dim3 grid1(nqb1 * a.Hkv, 1, a.n_splits);
    auto go2 = [&](auto kern, int smem) {
      smem_attr_once(kern, smem);
      launch_pdl(kern, grid1, dim3(576), smem, stream, tk, tv, at, G, nqb1);
      if (trace_path) {
        unsigned long long h[4 * 256 * 4];
        cudaMemcpyAsync(h, trace_dev, sizeof(h), cudaMemcpyDeviceToHost, stream);
        cudaStreamSynchronize(stream);
        if (FILE* f = std::fopen(trace_path, "ab")) {
          std::fwrite(h, sizeof(h), 1, f);
          std::fclose(f);
        }
      }
    };
    // FRAG_ATTN_QTM_POLY: every n-th exp pair on the FMA pipe (0 = MUFU only)
    static const int qpoly = [] {
      const char* v = std::getenv("FRAG_ATTN_QTM_POLY");
      return v ? std::atoi(v) : kQtmPoly;
    }();
    if (a.dh == 128) {
      switch (qpoly) {
        case 0: go2(attn_qtm_kernel<128, 0>, (int)qtm_smem<128>()); break;
        case 2: go2(attn_qtm_kernel<128, 2>, (int)qtm_smem<128>()); break;
        case 3: go2(attn_qtm_kernel<128, 3>, (int)qtm_smem<128>()); break;
        case 8: go2(attn_qtm_kernel<128, 8>, (int)qtm_smem<128>()); break;
        default: go2(attn_qtm_kernel<128, 4>, (int)qtm_smem<128>()); break;
      }
    } else {
      go2(attn_qtm_kernel<64, kQtmPoly>, (int)qtm_smem<64>());
    }
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
  }
  if (split_rows && a.dh == 128 && poly == 0) {
    threads = 576;
    go(attn_tc_kernel<128, 0, false, true>, (int)AttCfg<128>::SMEM);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
  }
  if (a.dh == 128) {
    constexpr int SM = (int)AttCfg<128>::SMEM;
    switch (poly) {
      case 4: go(attn_tc_kernel<128, 4>, SM); break;
      default: go(attn_tc_kernel<128, kDefaultPoly>, SM); break;
    }
  } else if (a.dh == 64) {
    go(attn_tc_kernel<64, kDefaultPoly>, (int)AttCfg<64>::SMEM);
  } else {
    return -1;
  }
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace fragk
