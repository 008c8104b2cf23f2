// K4/K7/K8 at large M: CTA-pair (cta_group::2) tcgen05 GEMM.
//
//   C[M,N] = A[M,K] . B[N,K]^T, one 256 x BN output tile per CTA pair.
//
// A thread-block cluster of two CTAs on one TPC shares every MMA:
//   * each CTA TMA-loads its own 128 rows of A and its own BN/2 rows of B per
//     64-wide K step (SWIZZLE_128B), completing on the LEADER's full barrier;
//   * the leader's single MMA thread issues tcgen05.mma.cta_group::2 with
//     M=256, N=BN, K=16: the tensor cores of both SMs read A from their own
//     SM and B halves from both, so each SM moves half the B bytes of the
//     1-CTA kernel (96 -> 64 B/clk of shared-memory operand traffic at BN=256);
//   * commits are multicast to both CTAs' barriers; each CTA's epilogue reads
//     its own 128 accumulator lanes from TMEM and arrives remotely on the
//     leader's TMEM-empty barrier.
// Accumulators are double-buffered in TMEM (2 x BN columns per CTA) and the
// tile loop is persistent over CTA pairs. Epilogues are the ones of the 1-CTA
// kernel (gemm_epi.cuh).
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "gemm_epi.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace fragk {

namespace {

constexpr int BM2 = 256;  // rows per CTA pair
constexpr int BK2 = 64;
constexpr int GEMM2_THREADS = 192;
constexpr uint32_t PEER_MASK = 0xFEFFFFFFu;  // shared::cluster address of the same offset in CTA rank 0

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const void* tmap, uint32_t leader_bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(leader_bar), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  const uint16_t mask = 0x3;
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* smem_dst) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS) : "memory");
}

// tooling (FRAG_GEMM2_TRACE=<file>, tools/gemm2_trace.py): globaltimer stamps
// per CTA into ep.trace[cta][32]: 0 entry, 1 prologue done, 2 producer past the
// PDL wait, 4 + 4t + {0 first MMA, 1 last MMA issued, 2 accumulator seen by the
// epilogue, 3 epilogue done} for the CTA's t-th tile (t < 6), 30 exit
__device__ __forceinline__ void g2_stamp(const EpiParams& ep, int slot) {
  if (ep.trace) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    ep.trace[blockIdx.x * 32 + slot] = t;
  }
}

template <int BN>
struct Gemm2Cfg {
  static constexpr int STAGES = 6;
  static constexpr uint32_t A_BYTES = 128 * BK2 * 2;       // this CTA's 128 rows of A
  static constexpr uint32_t B_BYTES = (BN / 2) * BK2 * 2;  // this CTA's BN/2 rows of B
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN <= 256 ? 256 : 512;
  static constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE_BYTES + 256;  // + barriers, TMEM slot, flag
  static_assert(SMEM <= 232448, "GEMM pipeline exceeds the 227 KB shared-memory limit");
};

template <int BN, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GEMM2_THREADS, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                    int K, const EpiParams ep) {
  using C = Gemm2Cfg<BN>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * C::B_BYTES);  // used in the leader
  uint64_t* empty = full + STAGES;                                           // both CTAs (multicast)
  uint64_t* tfull = empty + STAGES;                                          // both CTAs (multicast)
  uint64_t* tempty = tfull + 2;                                              // used in the leader
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  const int m_tiles = (M + BM2 - 1) / BM2;
  const int n_tiles = (N + BN - 1) / BN;  // last N tile may be partial (BN = 192, 224)
  const int num_tiles = m_tiles * n_tiles;
  const int nk = K / BK2;
  // work items: the first n_full tiles whole, then each tail tile cut into
  // `splits` K ranges (split-K of the last partial wave); the split CTAs of
  // each 128-row half-tile reduce it cooperatively (split_fixup)
  const int splits = ep.splits > 1 ? ep.splits : 1;
  const int n_full = splits > 1 ? ep.full_tiles : num_tiles;
  const int num_work = n_full + (num_tiles - n_full) * splits;
  // tile -> (m_blk, n_blk): groups of GM M-blocks, M fastest inside a group
  // (GM = m_tiles: plain M-fastest order)
  const int GM = ep.group_m > 0 && ep.group_m < m_tiles ? ep.group_m : m_tiles;
  auto tile_mn = [&](int t, int& mb, int& nb) {
    const int per_group = GM * n_tiles;
    const int g = t / per_group, idx = t - g * per_group;
    const int gm = min(GM, m_tiles - g * GM);
    mb = g * GM + idx % gm;
    nb = idx / gm;
  };
  auto decode = [&](int w, int& tile, int& sp, int& S) {
    if (w < n_full) {
      tile = w, sp = 0, S = 1;
    } else {
      const int u = w - n_full;
      tile = n_full + u / splits, sp = u % splits, S = splits;
    }
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 2);  // leader's expect_tx arrive + the peer's remote arrive
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // 4 epilogue warps x 2 CTAs
    }
    fence_mbar_init();
  }
  if (threadIdx.x == 0) g2_stamp(ep, 0);
  if (warp == 1) tmem_alloc_pair<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) g2_stamp(ep, 1);

  if (warp == 0) {
    if (elect_one()) {
      pdl_launch_dependents();
      // weight (B) loads of the first stages go out before the dependency wait
      int npre = 0;
      if (pair < num_work) {
        int tile, sp, S;
        decode(pair, tile, sp, S);
        int m_blk, n_blk;
        tile_mn(tile, m_blk, n_blk);
        const int kb0 = sp * nk / S, kb1 = (sp + 1) * nk / S;
        npre = kb1 - kb0 < STAGES ? kb1 - kb0 : STAGES;
        for (int i = 0; i < npre; ++i) {
          const uint32_t fb = smem_u32(&full[i]) & PEER_MASK;
          if (leader)
            mbar_arrive_expect_tx(&full[i], 2 * C::STAGE_BYTES);
          else
            mbar_arrive_cluster(fb);
          tma_load_2d_pair(sB + i * C::B_BYTES, &tmB, fb, (kb0 + i) * BK2, n_blk * BN + rank * (BN / 2));
        }
      }
      pdl_wait();
      g2_stamp(ep, 2);
      int stage = 0, it = 0;
      uint32_t phase = 0;
      for (int w = pair; w < num_work; w += n_pairs) {
        int tile, sp, S;
        decode(w, tile, sp, S);
        int m_blk, n_blk;
        tile_mn(tile, m_blk, n_blk);
        const int kb0 = sp * nk / S, kb1 = (sp + 1) * nk / S;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const uint32_t fb = smem_u32(&full[stage]) & PEER_MASK;
          if (it >= npre) {
            mbar_wait(&empty[stage], phase ^ 1);
            if (leader)
              mbar_arrive_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
            else
              mbar_arrive_cluster(fb);
            tma_load_2d_pair(sB + stage * C::B_BYTES, &tmB, fb, kb * BK2, n_blk * BN + rank * (BN / 2));
          }
          tma_load_2d_pair(sA + stage * C::A_BYTES, &tmA, fb, kb * BK2, m_blk * BM2 + rank * 128);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM2, BN, 0, 0);
      const uint64_t da = umma_desc_sw128(smem_u32(sA), 16, 1024);
      const uint64_t db = umma_desc_sw128(smem_u32(sB), 16, 1024);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int tcount = 0;
      for (int w = pair; w < num_work; w += n_pairs, ++tcount) {
        int tile, sp, S;
        decode(w, tile, sp, S);
        const int kb0 = sp * nk / S, kb1 = (sp + 1) * nk / S;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        if (tcount < 6 && lane == 0) g2_stamp(ep, 4 + 4 * tcount);
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t a0 = da + ((stage * C::A_BYTES) >> 4);
            const uint64_t b0 = db + ((stage * C::B_BYTES) >> 4);
#pragma unroll
            for (int k = 0; k < BK2 / 16; ++k)
              umma_bf16_pair(d_tmem, a0 + 2 * k, b0 + 2 * k, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
            umma_commit_pair(&empty[stage]);
            if (kb == kb1 - 1) umma_commit_pair(&tfull[acc]);
            if (kb == kb1 - 1 && tcount < 6) g2_stamp(ep, 5 + 4 * tcount);
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    pdl_wait();  // the epilogue reads/writes buffers of the preceding kernels
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row_in_tile = q * 32 + lane;
    const uint32_t te_leader = smem_u32(tempty) & PEER_MASK;
    int acc = 0;
    uint32_t acc_phase = 0;
    int tcount = 0;
    for (int w = pair; w < num_work; w += n_pairs, ++tcount) {
      int tile, sp, S;
      decode(w, tile, sp, S);
      int m_blk, n_blk;
      tile_mn(tile, m_blk, n_blk);
      const int row = m_blk * BM2 + rank * 128 + row_in_tile;
      // folded RMSNorm scale, loaded while the MMAs run
      const float rs = row < M ? epi_row_scale<EPI>(ep, row) : 1.f;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if (warp == 2 && lane == 0 && tcount < 6) g2_stamp(ep, 6 + 4 * tcount);
      const uint32_t t_row = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      if (S == 1) {
        if constexpr (EPI == EPI_SWIGLU) {
#pragma unroll 1
          for (int c = 0; c < BN / 32; c += 2) {
            uint32_t r[32], r2[32];
            tmem_ld32(t_row + c * 32, r);
            tmem_ld32(t_row + (c + 1) * 32, r2);
            tmem_ld_wait();
            if (row < M && n_blk * BN + c * 32 < N) epi_chunk<EPI>(ep, row, n_blk * BN + c * 32, r, r2, rs);
          }
        } else {
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(t_row + c * 32, r);
            tmem_ld_wait();
            if (row < M && n_blk * BN + c * 32 < N) epi_chunk<EPI>(ep, row, n_blk * BN + c * 32, r, r, rs);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(te_leader + acc * 8);
        if (warp == 2 && lane == 0 && tcount < 6) g2_stamp(ep, 7 + 4 * tcount);
      } else {
        // split partial of this CTA's 128 rows -> workspace (fp32); TMEM freed at once
        const int slot = (tile - n_full) * 2 + (int)rank;  // counter / workspace half-tile slot
        float* wsp = ep.ws + ((size_t)(slot * S + sp) * 128 + row_in_tile) * BN;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(t_row + c * 32, r);
          tmem_ld_wait();
          float4* dst = reinterpret_cast<float4*>(wsp + c * 32);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            dst[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                 __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(te_leader + acc * 8);
        split_fixup<BN, EPI>(ep, slot, S, sp, 128, row_in_tile, row, M, n_blk * BN, warp == 2 && lane == 0, rs);
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  tc_fence_before();
  cluster_sync();
  if (threadIdx.x == 0) g2_stamp(ep, 30);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair<C::TMEM_COLS>(tmem_base);
  }
}

template <int BN, int EPI>
int launch2(const bf16* A, const bf16* B, int M, int N, int K, const EpiParams& ep0, cudaStream_t stream) {
  using C = Gemm2Cfg<BN>;
  static const int group_env = [] {  // FRAG_GEMM_GROUP_M: tile raster, M blocks per group (tuning)
    const char* v = std::getenv("FRAG_GEMM_GROUP_M");
    return v ? std::atoi(v) : 0;
  }();
  EpiParams ep = ep0;
  if (group_env > 0) ep.group_m = group_env;
  smem_attr_once(gemm_tc2_kernel<BN, EPI>, (int)C::SMEM);
  CUtensorMap ta, tb;
  if (!make_tmap_2d(&ta, A, M, K, K, 128)) return -1;
  if (!make_tmap_2d(&tb, B, N, K, K, BN / 2)) return -1;
  const int tiles = ((M + BM2 - 1) / BM2) * ((N + BN - 1) / BN);
  const int work = ep.splits > 1 ? ep.full_tiles + (tiles - ep.full_tiles) * ep.splits : tiles;
  const int pairs = num_sms() / 2;
  const int grid = 2 * (work < pairs ? work : pairs);
  if (ep.splits > 1 && grid > num_sms() * resident_blocks(gemm_tc2_kernel<BN, EPI>, GEMM2_THREADS, (int)C::SMEM))
    return -1;  // the tail split's fixup waits on other CTAs of the grid
  static const char* trace_path = std::getenv("FRAG_GEMM2_TRACE");  // tooling (tools/gemm2_trace.py)
  static unsigned long long* trace_dev = nullptr;
  if (trace_path) {
    if (!trace_dev) cudaMalloc(&trace_dev, 160 * 32 * sizeof(unsigned long long));
    cudaMemsetAsync(trace_dev, 0, 160 * 32 * sizeof(unsigned long long), stream);
    ep.trace = trace_dev;
  }
  launch_pdl(gemm_tc2_kernel<BN, EPI>, dim3(grid), dim3(GEMM2_THREADS), C::SMEM, stream, ta, tb, M, N, K, ep);
  if (trace_path) {
    std::vector<unsigned long long> h(160 * 32);
    cudaMemcpyAsync(h.data(), trace_dev, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream);
    cudaStreamSynchronize(stream);
    if (FILE* f = std::fopen(trace_path, "ab")) {
      std::fwrite(h.data(), sizeof(unsigned long long), h.size(), f);
      std::fclose(f);
    }
  }
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace

// Large-M GEMM on CTA pairs (BN = 256 or 128 per pair). Returns launches or -1.
namespace {
int pair_dispatch(const bf16* A, const bf16* B, int M, int N, int K, EpiKind epi, const EpiParams& ep,
                  cudaStream_t s, int bn);
}

int gemm_bf16_tc_pair(const bf16* A, const bf16* B, int M, int N, int K, EpiKind epi, const EpiParams& ep,
                      cudaStream_t s, int bn, bool tail_split) {
  if (K % BK2 != 0 || N % 64 != 0 || (bn != 192 && bn != 224 && N % bn != 0)) return -1;
  if (bn == 224 && epi == EPI_SWIGLU) return -1;
  EpiParams ep2 = ep;
  ep2.splits = 1;
  if (!ep2.fault) ep2.fault = fault_slot_current();
  ep2.spin_ns = spin_limit_ns();
  if (tail_split && N % bn == 0 && ep.ws && ep.counters) {
    // split-K only the last partial wave of CTA pairs (deterministic reduction
    // per 128-row half by the last-arriving CTA)
    const long tiles = (long)((M + BM2 - 1) / BM2) * ((N + bn - 1) / bn), pairs = num_sms() / 2, nk = K / BK2;
    const long rem = tiles % pairs;
    long sp = rem ? pairs / rem : 1;
    if (sp > 8) sp = 8;
    while (sp > 1 && nk / sp < 4) --sp;
    if (sp > 1 && 2 * rem <= ep.counters_cap && (size_t)rem * 2 * sp * 128 * bn * sizeof(float) <= ep.ws_bytes) {
      ep2.splits = (int)sp;
      ep2.full_tiles = (int)(tiles - rem);
    }
  }
  return pair_dispatch(A, B, M, N, K, epi, ep2, s, bn);
}

namespace {
int pair_dispatch(const bf16* A, const bf16* B, int M, int N, int K, EpiKind epi, const EpiParams& ep,
                  cudaStream_t s, int bn) {
  if (bn == 256) {
    switch (epi) {
      case EPI_STORE_BF16: return launch2<256, EPI_STORE_BF16>(A, B, M, N, K, ep, s);
      case EPI_STORE_F32: return launch2<256, EPI_STORE_F32>(A, B, M, N, K, ep, s);
      case EPI_RESID: return launch2<256, EPI_RESID>(A, B, M, N, K, ep, s);
      case EPI_SWIGLU: return launch2<256, EPI_SWIGLU>(A, B, M, N, K, ep, s);
      case EPI_QKV: return launch2<256, EPI_QKV>(A, B, M, N, K, ep, s);
    }
  } else if (bn == 192) {
    switch (epi) {
      case EPI_STORE_BF16: return launch2<192, EPI_STORE_BF16>(A, B, M, N, K, ep, s);
      case EPI_STORE_F32: return launch2<192, EPI_STORE_F32>(A, B, M, N, K, ep, s);
      case EPI_RESID: return launch2<192, EPI_RESID>(A, B, M, N, K, ep, s);
      case EPI_SWIGLU: return launch2<192, EPI_SWIGLU>(A, B, M, N, K, ep, s);
      case EPI_QKV: return launch2<192, EPI_QKV>(A, B, M, N, K, ep, s);
    }
  } else if (bn == 224) {  // not SWIGLU: its gate/up column pairs are 64-aligned
    switch (epi) {
      case EPI_STORE_BF16: return launch2<224, EPI_STORE_BF16>(A, B, M, N, K, ep, s);
      case EPI_STORE_F32: return launch2<224, EPI_STORE_F32>(A, B, M, N, K, ep, s);
      case EPI_RESID: return launch2<224, EPI_RESID>(A, B, M, N, K, ep, s);
      case EPI_QKV: return launch2<224, EPI_QKV>(A, B, M, N, K, ep, s);
      default: return -1;
    }
  } else if (bn == 128) {
    switch (epi) {
      case EPI_STORE_BF16: return launch2<128, EPI_STORE_BF16>(A, B, M, N, K, ep, s);
      case EPI_STORE_F32: return launch2<128, EPI_STORE_F32>(A, B, M, N, K, ep, s);
      case EPI_RESID: return launch2<128, EPI_RESID>(A, B, M, N, K, ep, s);
      case EPI_SWIGLU: return launch2<128, EPI_SWIGLU>(A, B, M, N, K, ep, s);
      case EPI_QKV: return launch2<128, EPI_QKV>(A, B, M, N, K, ep, s);
    }
  }
  return -1;
}
}  // namespace

}  // namespace fragk
