// Weight-streaming GEMM chain for M <= 128 rows (question pass, decode): the
// per-layer projection sequence  O -> gate/up -> down -> next layer's QKV
// (K7, K8, K8, K4+K5 of SPEC.md:435-444 at |Q| rows) in ONE persistent launch.
//
// Each op is the same computation as gemm_tc_kernel<128, EPI, AR> (A = the
// live AR >= M activation rows, B = the weights, BN = 128, deterministic split-K
// with the cooperative fixup of gemm_epi.cuh) -- the chain only removes the
// kernel boundaries: the TMA ring, the TMEM accumulators and the CTAs stay
// alive from one op to the next, so op i+1's weights stream into the ring
// while op i's last MMAs, split-K fixups and epilogues finish. Op i+1's A
// operand is op i's output: its TMA loads wait on op i's completion counter
// (release/acquire + async-proxy fence), everything else (weights, TMEM,
// barriers) runs ahead.
//
// All CTAs are co-resident (one per SM, grid = #SMs), so spinning on another
// CTA's progress cannot deadlock; the counters are zero at launch and the last
// CTA out resets them.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "attn_combine.cuh"
#include "gemm_epi.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace fragk {

namespace {

constexpr int CBM = 128;  // UMMA M (accumulator rows; rows >= M are never stored)
constexpr int CBN = 128;
constexpr int CBK = 64;
// ring depth at <= 32 rows: 11 x 20 KB fills the 227 KB of shared memory with
// the static epilogue scratch (10 -> 11 measured within noise, kept; a build
// override for A/Bs)
#ifndef CHAIN_STAGES32
#define CHAIN_STAGES32 11
#endif
// AR = live A rows loaded per stage (32 / 64 / 128: M <= AR); stage = AR x 64
// activations + 128 x 64 weights, as many stages as fit in shared memory
template <int AR>
struct ChainCfg {
  static constexpr uint32_t A_BYTES = AR * 64 * 2;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + 128 * 64 * 2;
  static constexpr int STAGES = AR == 32 ? CHAIN_STAGES32 : (AR == 64 ? 8 : 6);
  static constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE_BYTES + 256;
  static_assert(STAGE_BYTES >= 128 * 64 * 2, "aliased A rows must stay inside the stage");
  static_assert(SMEM <= 232448, "chain ring exceeds the 227 KB shared-memory limit");
};
constexpr int CHAIN_THREADS = 192;
constexpr int CTMEM_COLS = 256;
constexpr int CHAIN_CNT_STRIDE = 512;  // fixup counter slots per op (tiles <= 512)                          // 2 x BN accumulators

struct ChainArgs {
  CUtensorMap tmA[CHAIN_MAX_OPS];
  CUtensorMap tmB[CHAIN_MAX_OPS];
  ChainOp op[CHAIN_MAX_OPS];
  int n_ops;
  int M;
  int* done;  // [CHAIN_MAX_OPS] op completion counters, [CHAIN_MAX_OPS] CTA exit counter,
              // [CHAIN_MAX_OPS + 1] pre-op (attention combine) completion
  AttnArgs pre;  // split-KV attention whose combine writes op 0's A operand
  int pre_rows;  // (token, head) rows to combine; 0 = no pre-op
  int timeline;  // tooling (FRAG_CHAIN_TRACE=1): globaltimer stamps into g_chain_tl
  int flow;      // 1: units continue round-robin across ops and A loads wait per producer tile
};


// Tooling timeline, graph-replay safe: launch n writes ring slot n % TL_LAUNCHES
// (n = g_chain_seq, read after griddepcontrol.wait and bumped by the last CTA
// out); per CTA [0] entry, [1] PDL wait done, [2] exit, [8 + 8 op + k] op
// stamps k = A ready, loads issued, first accumulator, published, fixup
// partial written, fixup siblings arrived. Read by frag_debug_chain_timeline.
constexpr int TL_LAUNCHES = 64, TL_CTAS = 160, TL_SLOTS = 8 + 8 * CHAIN_MAX_OPS;
__device__ unsigned long long g_chain_tl[TL_LAUNCHES][TL_CTAS][TL_SLOTS];
__device__ int g_chain_seq;

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long* chain_tl(const ChainArgs& a) {
  if (!a.timeline || blockIdx.x >= TL_CTAS) return nullptr;
  const int n = *reinterpret_cast<volatile int*>(&g_chain_seq);
  return &g_chain_tl[n % TL_LAUNCHES][blockIdx.x][0];
}
__device__ __forceinline__ void chain_stamp(unsigned long long* tl, int o, int k) {
  if (tl) tl[8 + 8 * o + k] = gtime();
}

// bounded wait on a counter of this launch (ptx.cuh spin_until_ge); the fault
// slot and limit travel in every op's EpiParams (op 0's are used)
__device__ __forceinline__ void wait_count(const int* p, int target, const EpiParams& ep) {
  spin_until_ge(p, target, ep.fault, ep.spin_ns);
}
// release-increment without waiting for the result (the writer does not stall
// on the atomic's round trip); cumulative over the CTA's writes ordered before
// it by bar.sync
__device__ __forceinline__ void red_release(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void tstamp(unsigned long long* p) {
  if (p) *p = gtime();
}

// Split-K fixup of one chain op (cf. split_fixup in gemm_epi.cuh): every
// split CTA of the tile waits for all S partials and reduces its share of the
// 32-column chunks in split order (bit-identical to split_fixup). Each op has
// its own counter slots (reset by the chain's last CTA), so there is no second
// round of arrivals, and the arrival is a release-reduction (the writer does
// not wait for the atomic). Measured: the op's fixup time is unchanged -- it
// is dominated by the slowest sibling and the reduction's L2 round trips.
template <int EPI>
__device__ __forceinline__ void chain_fixup(const EpiParams& ep, int* cnt, int slot, int S, int sp, int M,
                                            int row_in_tile, int col0, bool leader, float rs,
                                            unsigned long long* ts) {
  asm volatile("bar.sync 1, 128;" ::: "memory");
  if (leader) {
    tstamp(ts ? ts + 4 : nullptr);
    red_release(cnt, 1);
    wait_count(cnt, S, ep);
    tstamp(ts ? ts + 5 : nullptr);
  }
  asm volatile("bar.sync 1, 128;" ::: "memory");
  const float* base = ep.ws + ((size_t)slot * S * M + row_in_tile) * CBN;
  if (row_in_tile < M) reduce_partials<CBN, EPI>(ep, base, (size_t)M * CBN, S, sp, S, row_in_tile, col0, rs);
}

// unit u of an op: N tile and k-blocks kb0 + i * ks, i < n_kb (split sp of S:
// a contiguous range, or with ep.k_strided the blocks sp, sp + S, ...)
__device__ __forceinline__ void chain_unit(const ChainOp& op, int u, int& tile, int& kb0, int& ks, int& n_kb,
                                           int& sp, int& S) {
  S = op.splits > 1 ? op.splits : 1;
  if (op.sp_major) {  // the CTAs dealt an op's first units get the lowest k-ranges
    const int tiles = op.N / CBN;
    sp = u / tiles, tile = u % tiles;
  } else {
    tile = u / S, sp = u % S;
  }
  const int nk = op.K / CBK;
  if (op.ep.k_strided && S > 1) {
    kb0 = sp, ks = S, n_kb = (nk - sp + S - 1) / S;
  } else {
    kb0 = sp * nk / S, ks = 1, n_kb = (sp + 1) * nk / S - kb0;
  }
}
__device__ __forceinline__ int chain_units(const ChainOp& op) {
  return (op.N / CBN) * (op.splits > 1 ? op.splits : 1);
}

// Units of op o run on CTAs (unit + base_o) % G, base_o = units of the
// earlier ops: one round-robin over the whole chain, so op o's first units
// land on the CTAs op o-1 left idle (its last partial wave). Per-tile
// completion counters of op o (tdone) let op o+1's A loads wait only for the
// producer tiles of their k-block: op o+1 streams weights and starts its MMAs
// while op o's tail, fixups and epilogues finish.
__device__ __forceinline__ int chain_first_unit(const ChainArgs& a, int o, int G) {
  if (!a.flow) return blockIdx.x;
  int base = 0;
  for (int i = 0; i < o; ++i) base += chain_units(a.op[i]);
  return ((int)blockIdx.x - base % G + G) % G;
}
__device__ __forceinline__ int* chain_tdone(const ChainArgs& a, int o) {
  return a.op[o].ep.counters + (CHAIN_MAX_OPS + o) * CHAIN_CNT_STRIDE;
}

// Epilogue of one unit (4 warps, named barrier 1): direct fused epilogue, or
// the split partial + the cooperative deterministic fixup.
template <int EPI>
__device__ __forceinline__ void chain_epilogue(const EpiParams& ep, int* cnt, int M, int tile, int sp, int S,
                                               int row_in_tile, int q, int lane, int warp, uint32_t t_row,
                                               uint64_t* tempty_acc, float rs, unsigned long long* ts) {
  const int row = row_in_tile;  // one M tile
  const int col0 = tile * CBN;
  if (S <= 1) {
    if constexpr (EPI == EPI_SWIGLU) {
#pragma unroll 1
      for (int c = 0; c < CBN / 32; c += 2) {
        uint32_t r[32], r2[32];
        tmem_ld32(t_row + c * 32, r);
        tmem_ld32(t_row + (c + 1) * 32, r2);
        tmem_ld_wait();
        if (row < M) epi_chunk<EPI>(ep, row, col0 + c * 32, r, r2, rs);
      }
    } else {
#pragma unroll 1
      for (int c = 0; c < CBN / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(t_row + c * 32, r);
        tmem_ld_wait();
        if (row < M) epi_chunk<EPI>(ep, row, col0 + c * 32, r, r, rs);
      }
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(tempty_acc);
  } else {
    float* wsp = ep.ws + ((size_t)(tile * S + sp) * M + row_in_tile) * CBN;
#pragma unroll 1
    for (int c = 0; c < CBN / 32; ++c) {
      uint32_t r[32];
      tmem_ld32(t_row + c * 32, r);
      tmem_ld_wait();
      if (row_in_tile < M) {
        float4* dst = reinterpret_cast<float4*>(wsp + c * 32);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          dst[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                               __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
      }
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(tempty_acc);
    chain_fixup<EPI>(ep, cnt + tile, tile, S, sp, M, row_in_tile, col0, warp == 2 && lane == 0, rs, ts);
  }
}

template <int AR>
__global__ void __launch_bounds__(CHAIN_THREADS, 1) gemm_chain_kernel(const __grid_constant__ ChainArgs args) {
  constexpr int CSTAGES = ChainCfg<AR>::STAGES;
  constexpr uint32_t CA_BYTES = ChainCfg<AR>::A_BYTES;
  constexpr uint32_t CSTAGE_BYTES = ChainCfg<AR>::STAGE_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + CA_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + CSTAGES * CSTAGE_BYTES);
  uint64_t* empty = full + CSTAGES;
  uint64_t* tfull = empty + CSTAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_id();
  const int lane = lane_id();
  const int G = gridDim.x;
  const int n_ops = args.n_ops;
  const int M = args.M;

  if (warp == 0 && lane == 0) {
    for (int o = 0; o < n_ops; ++o) {
      tma_prefetch_desc(&args.tmA[o]);
      tma_prefetch_desc(&args.tmB[o]);
    }
    for (int s = 0; s < CSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<CTMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    // lane 0 issues; with flow the whole warp polls the A producer tiles
    const unsigned long long t_entry = gtime();
    unsigned long long* tl = nullptr;
    if (lane == 0) pdl_launch_dependents();
    int stage = 0;
    uint32_t phase = 0;
    auto advance = [&]() {
      if (++stage == CSTAGES) stage = 0, phase ^= 1;
    };
    for (int o = 0; o < n_ops; ++o) {
      const ChainOp& op = args.op[o];
      const CUtensorMap* tA = &args.tmA[o];
      const CUtensorMap* tB = &args.tmB[o];
      const int units = chain_units(op);
      const int u0 = chain_first_unit(args, o, G);
      // weights first: the first unit's leading stages, before waiting on
      // the op that produces this op's A rows
      int npre = 0, st_pre = stage;
      int tile, kb0, ks, n_kb, sp, S;
      if (u0 < units) {
        chain_unit(op, u0, tile, kb0, ks, n_kb, sp, S);
        npre = n_kb < CSTAGES ? n_kb : CSTAGES;
        for (int i = 0; i < npre; ++i) {
          if (lane == 0) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_arrive_expect_tx(&full[stage], CSTAGE_BYTES);
            tma_load_2d(sB + stage * CSTAGE_BYTES, tB, &full[stage], (kb0 + i * ks) * CBK, tile * CBN);
          }
          advance();
        }
      }
      if (o == 0) {
        pdl_wait();  // every CTA, before it reads any counter of this launch
        if (lane == 0) {
          tl = chain_tl(args);
          if (tl) tl[0] = t_entry, tl[1] = gtime();
        }
      }
      if (u0 >= units) continue;
      // A readiness: op 0 -- the in-chain combine (all CTAs); op o > 0 -- with
      // flow, the producer tile of each k-block (SWIGLU: one tile per 64 act
      // columns; RESID: one per 128 x columns), polled 32 tiles at a time;
      // without flow, every unit of op o-1
      const ChainOp* prev = o > 0 ? &args.op[o - 1] : nullptr;
      const int* ptd = o > 0 ? chain_tdone(args, o - 1) : nullptr;
      const int p_tiles = o > 0 ? prev->N / CBN : 0;
      const int p_need = o > 0 ? (prev->splits > 1 ? prev->splits : 1) : 0;
      const bool p_swiglu = o > 0 && prev->epi == EPI_SWIGLU;
      int win_base = -64;
      unsigned win_mask = 0u;
      auto a_ready = [&](int kb) {
        if (o == 0 || !args.flow) return;
        const int pt = p_swiglu ? kb : (kb >> 1);
        const int off = pt - win_base;
        if (off >= 0 && off < 32 && ((win_mask >> off) & 1u)) return;
        for (;;) {
          win_base = pt;
          const int t = pt + lane;
          const bool ok = t >= p_tiles || ld_acquire_gpu(ptd + t) >= p_need;
          win_mask = __ballot_sync(0xffffffffu, ok);
          if (win_mask & 1u) break;
          if (lane == 0) wait_count(ptd + pt, p_need, args.op[0].ep);
          __syncwarp();
        }
        __syncwarp();  // orders the lanes' acquires before lane 0's loads
        if (lane == 0) asm volatile("fence.proxy.async.global;" ::: "memory");  // generic writes -> TMA reads
      };
      if (lane == 0) {
        if (o == 0) {
          if (args.pre_rows > 0) {  // op 0's A rows come from the in-chain combine
            wait_count(&args.done[CHAIN_MAX_OPS + 1], G, args.op[0].ep);
            asm volatile("fence.proxy.async.global;" ::: "memory");
          }
        } else if (!args.flow) {
          wait_count(&args.done[o - 1], chain_units(args.op[o - 1]), args.op[0].ep);
          asm volatile("fence.proxy.async.global;" ::: "memory");  // generic writes -> TMA reads
        }
      }
      __syncwarp();
      if (lane == 0) chain_stamp(tl, o, 0);
      for (int i = 0, s2 = st_pre; i < npre; ++i, s2 = s2 + 1 == CSTAGES ? 0 : s2 + 1) {
        a_ready(kb0 + i * ks);
        if (lane == 0) tma_load_2d(sA + s2 * CSTAGE_BYTES, tA, &full[s2], (kb0 + i * ks) * CBK, 0);
      }
      for (int i = npre; i < n_kb; ++i) {
        const int kb = kb0 + i * ks;
        a_ready(kb);
        if (lane == 0) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], CSTAGE_BYTES);
          tma_load_2d(sB + stage * CSTAGE_BYTES, tB, &full[stage], kb * CBK, tile * CBN);
          tma_load_2d(sA + stage * CSTAGE_BYTES, tA, &full[stage], kb * CBK, 0);
        }
        advance();
      }
      for (int u = u0 + G; u < units; u += G) {
        chain_unit(op, u, tile, kb0, ks, n_kb, sp, S);
        for (int i = 0; i < n_kb; ++i) {
          const int kb = kb0 + i * ks;
          a_ready(kb);
          if (lane == 0) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_arrive_expect_tx(&full[stage], CSTAGE_BYTES);
            tma_load_2d(sB + stage * CSTAGE_BYTES, tB, &full[stage], kb * CBK, tile * CBN);
            tma_load_2d(sA + stage * CSTAGE_BYTES, tA, &full[stage], kb * CBK, 0);
          }
          advance();
        }
      }
      if (lane == 0) chain_stamp(tl, o, 1);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = umma_idesc_bf16(CBM, CBN, 0, 0);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int o = 0; o < n_ops; ++o) {
      const ChainOp& op = args.op[o];
      const int units = chain_units(op);
      for (int u = chain_first_unit(args, o, G); u < units; u += G) {
        int tile, kb0, ks, n_kb, sp, S;
        chain_unit(op, u, tile, kb0, ks, n_kb, sp, S);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * CBN;
        for (int i = 0; i < n_kb; ++i) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t a_base = smem_u32(sA + stage * CSTAGE_BYTES);
            const uint32_t b_base = smem_u32(sB + stage * CSTAGE_BYTES);
#pragma unroll
            for (int k = 0; k < CBK / 16; ++k) {
              const uint64_t ad = umma_desc_sw128(a_base + k * 32, 16, 1024);
              const uint64_t bd = umma_desc_sw128(b_base + k * 32, 16, 1024);
              umma_bf16_ss(d_tmem, ad, bd, idesc, (i != 0 || k != 0) ? 1u : 0u);
            }
            umma_commit(&empty[stage]);
            if (i == n_kb - 1) umma_commit(&tfull[acc]);
          }
          __syncwarp();
          if (++stage == CSTAGES) stage = 0, phase ^= 1;
        }
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..5)
    pdl_wait();
    __shared__ float rs_part[4][32];  // cooperative RMSNorm scale (M <= 32)
    unsigned long long* tl = (warp == 2 && lane == 0) ? chain_tl(args) : nullptr;
    const int q = warp & 3;
    const int row_in_tile = q * 32 + lane;
    if (args.pre_rows > 0) {
      // pre-op: merge the attention's split-KV partials into op 0's A rows,
      // one warp per (token, head) row, then publish (every CTA counts once)
      const size_t step = (size_t)G * 4;
      for (size_t qi = (size_t)blockIdx.x * 4 + q; qi < (size_t)args.pre_rows; qi += 2 * step) {
        const bool has_b = qi + step < (size_t)args.pre_rows;
        if (args.pre.dh == 128)
          attn_combine_row2<128>(args.pre, qi, qi + step, has_b, lane);
        else
          attn_combine_row2<64>(args.pre, qi, qi + step, has_b, lane);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (warp == 2 && lane == 0) red_release(&args.done[CHAIN_MAX_OPS + 1], 1);
    }
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int o = 0; o < n_ops; ++o) {
      const ChainOp& op = args.op[o];
      const int units = chain_units(op);
      const int u0 = chain_first_unit(args, o, G);
      if (u0 >= units) continue;
      // this op's epilogue reads / writes what the earlier ops of the chain wrote
      if (o > 0) wait_count(&args.done[o - 1], chain_units(args.op[o - 1]), args.op[0].ep);
      if (o > 1) wait_count(&args.done[o - 2], chain_units(args.op[o - 2]), args.op[0].ep);
      const EpiParams& ep = op.ep;
      int* cnt = ep.counters + o * CHAIN_CNT_STRIDE;  // this op's fixup counters
      unsigned long long* ts = tl ? tl + 8 + 8 * o : nullptr;
      float rs = 1.f;
      const bool need_rs = (op.epi == EPI_QKV || op.epi == EPI_SWIGLU) && ep.ssq_in;
      if (need_rs && M <= 32 && (ep.ssq_n & 3) == 0 && ep.ssq_n <= 4 * 32) {
        // rows live in warp 0 only: the four epilogue warps each take one of
        // epi_row_scale's four running sums (chunks w, w+4, ... in order, all
        // loads in flight at once, from L2), combined in its order -> same bits
        const int row = lane;
        float sw = 0.f;
        if (row < M) {
          const float* p = ep.ssq_in + row;
          const size_t ld = (size_t)ep.ssq_ld;
          float v[32];
#pragma unroll
          for (int k = 0; k < 32; ++k) v[k] = (q + 4 * k < ep.ssq_n) ? __ldcg(p + (q + 4 * k) * ld) : 0.f;
#pragma unroll
          for (int k = 0; k < 32; ++k)
            if (q + 4 * k < ep.ssq_n) sw += v[k];
        }
        rs_part[q][lane] = sw;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (q == 0 && row < M)
          rs = rsqrtf(((rs_part[0][row] + rs_part[1][row]) + (rs_part[2][row] + rs_part[3][row])) /
                          (float)ep.norm_d + ep.norm_eps);
        asm volatile("bar.sync 1, 128;" ::: "memory");  // rs_part reusable by the next op
      } else if (row_in_tile < M) {
        switch (op.epi) {
          case EPI_QKV: rs = epi_row_scale<EPI_QKV>(ep, row_in_tile); break;
          case EPI_SWIGLU: rs = epi_row_scale<EPI_SWIGLU>(ep, row_in_tile); break;
          default: break;
        }
      }
      for (int u = u0; u < units; u += G) {
        int tile, kb0, ks, n_kb, sp, S;
        chain_unit(op, u, tile, kb0, ks, n_kb, sp, S);
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        if (u == u0) chain_stamp(tl, o, 2);
        const uint32_t t_row = tmem_base + ((uint32_t)(q * 32) << 16) + acc * CBN;
        switch (op.epi) {
          case EPI_RESID:
            chain_epilogue<EPI_RESID>(ep, cnt, M, tile, sp, S, row_in_tile, q, lane, warp, t_row, &tempty[acc], rs, ts);
            break;
          case EPI_SWIGLU:
            chain_epilogue<EPI_SWIGLU>(ep, cnt, M, tile, sp, S, row_in_tile, q, lane, warp, t_row, &tempty[acc], rs, ts);
            break;
          case EPI_QKV:
            chain_epilogue<EPI_QKV>(ep, cnt, M, tile, sp, S, row_in_tile, q, lane, warp, t_row, &tempty[acc], rs, ts);
            break;
          default:
            chain_epilogue<EPI_STORE_BF16>(ep, cnt, M, tile, sp, S, row_in_tile, q, lane, warp, t_row, &tempty[acc],
                                           rs, ts);
            break;
        }
        // unit complete (its outputs written): publish the unit and its tile share
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (warp == 2 && lane == 0) {
          red_release(&args.done[o], 1);
          if (args.flow) red_release(chain_tdone(args, o) + tile, 1);
        }
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
      chain_stamp(tl, o, 3);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<CTMEM_COLS>(tmem_base);
  }
  if (threadIdx.x == 0) {
    if (unsigned long long* tl = chain_tl(args)) tl[2] = gtime();
    // the last CTA out re-arms the counters for the next launch (graph replay)
    int* exit_cnt = args.done + CHAIN_MAX_OPS;
    __threadfence();
    if (atomicAdd(exit_cnt, 1) == G - 1) {
      args.done[CHAIN_MAX_OPS + 1] = 0;
      for (int o = 0; o < n_ops; ++o) {
        args.done[o] = 0;
        const int tiles = args.op[o].N / CBN;
        int* cnt = args.op[o].ep.counters + o * CHAIN_CNT_STRIDE;
        int* td = chain_tdone(args, o);
        for (int t = 0; t < tiles; ++t) cnt[t] = 0, td[t] = 0;
      }
      *exit_cnt = 0;
      if (args.timeline) g_chain_seq = g_chain_seq + 1;
      __threadfence();
    }
  }
}

}  // namespace

bool gemm_chain_supported(int M, int N, int K) { return M >= 1 && M <= CBM && N % CBN == 0 && K % CBK == 0; }

int gemm_chain_tc(const ChainStep* steps, int n_ops, int M, int* done, cudaStream_t stream,
                  const AttnArgs* pre_combine) {
  if (n_ops < 1 || n_ops > CHAIN_MAX_OPS || !done) return -1;
  ChainArgs args{};
  if (pre_combine) {
    if (pre_combine->dh != 64 && pre_combine->dh != 128) return -1;
    args.pre = *pre_combine;
    args.pre_rows = pre_combine->M * pre_combine->Hq;
  }
  args.n_ops = n_ops;
  args.M = M;
  args.done = done;
  const long sms = num_sms();
  static const int sp_major = [] {  // FRAG_CHAIN_SPMAJOR=0: split units tile-major
    const char* v = std::getenv("FRAG_CHAIN_SPMAJOR");
    return v ? std::atoi(v) : 1;
  }();
  for (int o = 0; o < n_ops; ++o) {
    const ChainStep& st = steps[o];
    if (!gemm_chain_supported(M, st.N, st.K) || !st.ep.ws || !st.ep.counters) return -1;
    if (!make_tmap_2d(&args.tmA[o], st.A, M, st.K, st.K, M <= 32 ? 32 : (M <= 64 ? 64 : 128))) return -1;
    if (!make_tmap_2d(&args.tmB[o], st.B, st.N, st.K, st.K, CBN)) return -1;
    // the one-M-tile policy of gemm_bf16_tc: split-K up to one full wave (a
    // cost model that balanced the 224-tile gate/up with 5 splits and the
    // down projection with 9 -- several fixup rounds per op -- measured 47 %
    // slower: fixup waits that straddle rounds serialise)
    const long tiles = st.N / CBN, nk = st.K / CBK;
    long s = 1;
    while (s < 8 && tiles * (s + 1) <= sms && nk / (s + 1) >= 4) ++s;
    if (s > nk) s = nk;
    if ((size_t)(tiles * s * M * CBN) * sizeof(float) > st.ep.ws_bytes) s = 1;
    if (tiles > CHAIN_CNT_STRIDE || (CHAIN_MAX_OPS + o + 1) * CHAIN_CNT_STRIDE > st.ep.counters_cap) return -1;
    ChainOp& op = args.op[o];
    op.N = st.N;
    op.K = st.K;
    op.epi = st.epi;
    op.splits = (int)s;
    op.sp_major = sp_major;
    op.ep = st.ep;
    op.ep.splits = (int)s;
    op.ep.k_strided = s > 1 && k_strided_for(st.K / CBK) ? 1 : 0;  // same rule as gemm_bf16_tc
    op.ep.l2_reads = 1;
    if (!op.ep.fault) op.ep.fault = fault_slot_current();
    op.ep.spin_ns = spin_limit_ns();
    op.ep.full_tiles = 0;
    op.ep.streamk = 0;
  }
  static const bool timeline = std::getenv("FRAG_CHAIN_TRACE") != nullptr;  // tooling only
  args.timeline = timeline ? 1 : 0;
  static const bool flow = [] {  // FRAG_CHAIN_FLOW=0: per-op barriers, every op's units from CTA 0
    const char* v = std::getenv("FRAG_CHAIN_FLOW");
    return !(v && v[0] == '0');
  }();
  args.flow = flow ? 1 : 0;
  auto go = [&](auto kern, size_t smem) {
    smem_attr_once(kern, (int)smem);
    if (resident_blocks(kern, CHAIN_THREADS, (int)smem) < 1) return false;  // one CTA per SM must fit
    launch_pdl(kern, dim3((unsigned)sms), dim3(CHAIN_THREADS), smem, stream, args);
    return true;
  };
  bool ok;
  if (M <= 32)
    ok = go(gemm_chain_kernel<32>, ChainCfg<32>::SMEM);
  else if (M <= 64)
    ok = go(gemm_chain_kernel<64>, ChainCfg<64>::SMEM);
  else
    ok = go(gemm_chain_kernel<128>, ChainCfg<128>::SMEM);
  return ok && cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace fragk

// Tooling (tools/chain_trace.py; not part of the frag C API): copy the chain
// timeline ring. Returns the number of chain launches recorded so far.
extern "C" __attribute__((visibility("default"))) int frag_debug_chain_timeline(unsigned long long* out, int max_launches) {
  int seq = 0;
  cudaMemcpyFromSymbol(&seq, fragk::g_chain_seq, sizeof(int));
  const int n = max_launches < fragk::TL_LAUNCHES ? max_launches : fragk::TL_LAUNCHES;
  cudaMemcpyFromSymbol(out, fragk::g_chain_tl, (size_t)n * fragk::TL_CTAS * fragk::TL_SLOTS * 8);
  return seq;
}
