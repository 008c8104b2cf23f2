// K4/K7/K8/K11: persistent, warp-specialised tcgen05 GEMM for sm_100a.
//
//   C[M,N] = A[M,K] · B[N,K]^T     (A = activations, B = weights [out][in])
//
// Pipeline per CTA (one CTA per SM, 192 threads):
//   warp 0      TMA producer: A (128x64) and B (BNx64) tiles, SWIZZLE_128B,
//               into a STAGES-deep shared-memory ring guarded by mbarriers.
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//               (M=128, N=BN, K=16 per instruction), accumulator in TMEM,
//               double-buffered (2 x BN columns) so the epilogue of tile i
//               overlaps the MMAs of tile i+1.
//   warps 2..5  epilogue: tcgen05.ld 32x32b -> registers -> fused op -> global.
//
// The fused epilogues implement the projection-side work of the selective
// recompute (Eq. 9): RoPE at the global
// position + scatter of fresh K/V rows into the fused cache (K4+K5), residual
// add (K7, K8-down), SiLU(gate)*up (K8), fp32 logits (K11).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <unordered_map>

#include "gemm_epi.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace fragk {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // one 128-byte swizzle atom of bf16
constexpr int GEMM_THREADS = 192;

// AR = A rows loaded per stage (128, or 64 / 32 for the one-M-tile
// weight-streaming GEMMs). A stage is [A: AR rows][B: BN rows]; the UMMA still
// reads 128 A rows from the stage base, so rows AR..127 alias the stage's B
// bytes: they only feed accumulator rows >= M, which are never stored. Small
// stages leave room for a second CTA per SM (the next kernel's, under PDL).
template <int BN, int AR = BM>
struct GemmCfg {
  static constexpr int STAGES = AR < BM ? (AR == 32 ? 8 : 7) : (BN == 256 ? 4 : (BN == 128 ? 6 : 8));
  static constexpr int MIN_BLOCKS = 1;
  static constexpr uint32_t A_BYTES = AR * BK * 2;  // TMA bytes of A per stage
  static constexpr uint32_t B_BYTES = BN * BK * 2;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static_assert(STAGE_BYTES % 1024 == 0, "stages must stay 1024-byte aligned (SW128 atoms)");
  static_assert(AR == BM || STAGE_BYTES >= BM * BK * 2, "aliased A rows must stay inside the stage");
  static constexpr int TMEM_COLS = 2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512);
  static constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE_BYTES + 256;
  static_assert(SMEM <= 232448, "GEMM pipeline exceeds the 227 KB shared-memory limit");
};

template <int BN, int EPI, int AR = BM>
__global__ void __launch_bounds__(GEMM_THREADS, GemmCfg<BN, AR>::MIN_BLOCKS)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                   int K, const EpiParams ep) {
  using C = GemmCfg<BN, AR>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // stage s: A at smem + s*STAGE_BYTES, B right after it
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_id();
  const int lane = lane_id();
  const int m_tiles = (M + BM - 1) / BM;
  const int n_tiles = N / BN;
  const int num_tiles = m_tiles * n_tiles;
  const int nk = K / BK;

  auto stamp = [&](int k) {
    if (ep.trace && blockIdx.x < 256) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      ep.trace[blockIdx.x * 8 + k] = t;
    }
  };
  if (warp == 0 && lane == 0) {
    stamp(0);
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // Work decomposition, one of:
  //  * units: the first `full_tiles` tiles whole, then each tail tile cut into
  //    `splits` K ranges reduced cooperatively by its split CTAs (split_fixup);
  //  * stream-K (ep.streamk, one M tile): CTA c owns k-blocks
  //    [c*I/G, (c+1)*I/G) of the flattened (tile, k-block) space, I = tiles*nk,
  //    cut at tile boundaries into parts. A tile spread over several CTAs is
  //    finished by the CTA holding its first k-block (the "owner"): that part
  //    is the owner's last, while the other contributors' parts are their
  //    first, so the owner never waits on work that has not started; it sums
  //    the partials in CTA order (deterministic) and runs the epilogue.
  const bool sk = ep.streamk != 0;
  const int splits = ep.splits > 1 ? ep.splits : 1;
  const int n_full = splits > 1 ? ep.full_tiles : num_tiles;
  const int num_work = n_full + (num_tiles - n_full) * splits;
  const long long I = (long long)num_tiles * nk;
  const int G = gridDim.x;
  const long long sk_hi = sk ? I * (blockIdx.x + 1) / G : 0;
  auto first = [&]() -> long long { return sk ? I * blockIdx.x / G : (long long)blockIdx.x; };
  // next part: tile, split sp of S (S = 0 marks a stream-K part) and its
  // k-blocks kb0 + i * ks, i < n_kb: the range [kb0, kb1), or with
  // ep.k_strided the blocks sp, sp + S, ... (every split then holds an equal
  // share of the late-produced A columns, see the GEMM chain)
  auto next = [&](long long& st, int& tile, int& kb0, int& kb1, int& sp, int& S, int& ks, int& n_kb) -> bool {
    ks = 1;
    if (sk) {
      if (st >= sk_hi) return false;
      tile = (int)(st / nk);
      kb0 = (int)(st % nk);
      const long long left = sk_hi - st;
      kb1 = left < nk - kb0 ? kb0 + (int)left : nk;
      sp = 0, S = 0;
      st += kb1 - kb0;
      n_kb = kb1 - kb0;
      return true;
    }
    if (st >= num_work) return false;
    const int w = (int)st;
    if (w < n_full) {
      tile = w, sp = 0, S = 1;
    } else {
      const int u = w - n_full;
      tile = n_full + u / splits, sp = u % splits, S = splits;
    }
    if (ep.k_strided && S > 1) {
      kb0 = sp, kb1 = nk, ks = S, n_kb = (nk - sp + S - 1) / S;
    } else {
      kb0 = sp * nk / S, kb1 = (sp + 1) * nk / S, n_kb = kb1 - kb0;
    }
    st += G;
    return true;
  };
  if (warp == 0) {
    if (elect_one()) {
      pdl_launch_dependents();
      // Weights (B) do not depend on the preceding kernel: issue the first
      // stages' B loads before waiting on it (programmatic dependent launch),
      // then the activation (A) loads once its output is visible.
      int npre = 0;
      {
        long long st = first();
        int tile, kb0, kb1, sp, S, ks, n_kb;
        if (next(st, tile, kb0, kb1, sp, S, ks, n_kb)) {
          const int n_blk = tile / m_tiles;
          npre = n_kb < STAGES ? n_kb : STAGES;
          for (int i = 0; i < npre; ++i) {
            mbar_arrive_expect_tx(&full[i], C::STAGE_BYTES);
            tma_load_2d(sB + i * C::STAGE_BYTES, &tmB, &full[i], (kb0 + i * ks) * BK, n_blk * BN);
          }
        }
      }
      pdl_wait();
      stamp(1);
      int stage = 0, it = 0;
      uint32_t phase = 0;
      long long st = first();
      int tile, kb0, kb1, sp, S, ks, n_kb;
      while (next(st, tile, kb0, kb1, sp, S, ks, n_kb)) {
        const int m_blk = tile % m_tiles, n_blk = tile / m_tiles;
        for (int i = 0; i < n_kb; ++i, ++it) {
          const int kb = kb0 + i * ks;
          if (it >= npre) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
            tma_load_2d(sB + stage * C::STAGE_BYTES, &tmB, &full[stage], kb * BK, n_blk * BN);
          }
          tma_load_2d(sA + stage * C::STAGE_BYTES, &tmA, &full[stage], kb * BK, m_blk * BM);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = umma_idesc_bf16(BM, BN, 0, 0);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    long long st = first();
    int tile, kb0, kb1, sp, S, ks, n_kb;
    while (next(st, tile, kb0, kb1, sp, S, ks, n_kb)) {
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int i = 0; i < n_kb; ++i) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (i == 0 && lane == 0) stamp(2);
        if (elect_one()) {
          const uint32_t a_base = smem_u32(sA + stage * C::STAGE_BYTES);
          const uint32_t b_base = smem_u32(sB + stage * C::STAGE_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = umma_desc_sw128(a_base + k * 32, 16, 1024);
            const uint64_t bd = umma_desc_sw128(b_base + k * 32, 16, 1024);
            umma_bf16_ss(d_tmem, ad, bd, idesc, (i != 0 || k != 0) ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
          if (i == n_kb - 1) umma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (i == n_kb - 1 && lane == 0) stamp(3);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else {
    pdl_wait();  // the epilogue reads/writes buffers of the preceding kernels
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row_in_tile = q * 32 + lane;
    const int ws_rows = m_tiles == 1 ? M : BM;  // rows kept per split / stream-K partial
    int acc = 0;
    uint32_t acc_phase = 0;
    long long st = first();
    int tile, kb0, kb1, sp, S, ks, n_kb;
    while (next(st, tile, kb0, kb1, sp, S, ks, n_kb)) {
      const int m_blk = tile % m_tiles, n_blk = tile / m_tiles;
      const int ti = tile - n_full;  // tail index (workspace / counter slot)
      const int row = m_blk * BM + row_in_tile;
      // folded RMSNorm scale, loaded while the MMAs run
      const float rs = row < M ? epi_row_scale<EPI>(ep, row) : 1.f;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if (warp == 2 && lane == 0) stamp(4);
      const uint32_t t_row = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      if (S == 0 && !(kb0 == 0 && kb1 == nk)) {
        // stream-K part of a tile shared by several CTAs: partial -> workspace
        // slot (tile, CTA offset from the owner), TMEM released right away
        const long long p0 = (long long)tile * nk;
        const int c_own = sk_cta_of(p0, I, G);
        const int j = (int)blockIdx.x - c_own;
        float* wsp = ep.ws + (((size_t)tile * ep.sk_maxc + j) * ws_rows + row_in_tile) * BN;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(t_row + c * 32, r);
          tmem_ld_wait();
          if (row_in_tile < ws_rows) {
            float4* dst = reinterpret_cast<float4*>(wsp + c * 32);
#pragma unroll
            for (int e = 0; e < 8; ++e)
              __stcg(dst + e, make_float4(__uint_as_float(r[4 * e]), __uint_as_float(r[4 * e + 1]),
                                          __uint_as_float(r[4 * e + 2]), __uint_as_float(r[4 * e + 3])));
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        const int n_contrib = sk_cta_of(p0 + nk - 1, I, G) - c_own + 1;
        sk_finish<BN, EPI>(ep, tile, j, n_contrib, ws_rows, row_in_tile, row, M, n_blk * BN, warp == 2 && lane == 0,
                           rs);
      } else if (S <= 1) {
        if constexpr (EPI == EPI_SWIGLU) {
#pragma unroll 1
          for (int c = 0; c < BN / 32; c += 2) {
            uint32_t r[32], r2[32];
            tmem_ld32(t_row + c * 32, r);
            tmem_ld32(t_row + (c + 1) * 32, r2);
            tmem_ld_wait();
            if (row < M) epi_chunk<EPI>(ep, row, n_blk * BN + c * 32, r, r2, rs);
          }
        } else {
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(t_row + c * 32, r);
            tmem_ld_wait();
            if (row < M) epi_chunk<EPI>(ep, row, n_blk * BN + c * 32, r, r, rs);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      } else {
        // split partial -> workspace (fp32), TMEM released right away
        float* wsp = ep.ws + ((size_t)(ti * S + sp) * ws_rows + row_in_tile) * BN;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(t_row + c * 32, r);
          tmem_ld_wait();
          if (row_in_tile < ws_rows) {
            float4* dst = reinterpret_cast<float4*>(wsp + c * 32);
#pragma unroll
            for (int j = 0; j < 8; ++j)
              dst[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                   __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        if (warp == 2 && lane == 0) stamp(5);
        split_fixup<BN, EPI>(ep, ti, S, sp, ws_rows, row_in_tile, row, M, n_blk * BN, warp == 2 && lane == 0, rs);
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  if (warp == 2 && lane == 0) stamp(6);
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
}

// ----------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;
constexpr int kMaxDevices = 64;

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  std::call_once(g_encode_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode;
}

// 2-D bf16 tensor map over a row-major [rows][cols] matrix, box = box_rows x 64 cols.
}  // namespace

bool make_tmap_2d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t row_stride_elems,
                  uint32_t box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_stride_elems * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_tmap_3d(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1_elems,
                  uint64_t s2_elems, uint32_t b0, uint32_t b1, uint32_t b2) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1_elems * 2, s2_elems * 2};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

namespace {

template <int BN, int EPI, int AR = BM>
int launch(const bf16* A, const bf16* B, int M, int N, int K, const EpiParams& ep, cudaStream_t stream) {
  using C = GemmCfg<BN, AR>;
  smem_attr_once(gemm_tc_kernel<BN, EPI, AR>, (int)C::SMEM);
  CUtensorMap ta, tb;
  if (!make_tmap_2d(&ta, A, M, K, K, AR)) return -1;
  if (!make_tmap_2d(&tb, B, N, K, K, BN)) return -1;
  const int tiles = ((M + BM - 1) / BM) * (N / BN);
  const int work = ep.splits > 1 ? ep.full_tiles + (tiles - ep.full_tiles) * ep.splits : tiles;
  const int slots = num_sms() * C::MIN_BLOCKS;
  const int grid = ep.streamk ? ep.streamk : (work < slots ? work : slots);
  // split-K fixups / stream-K partial hand-offs wait on other CTAs of the grid
  if ((ep.splits > 1 || ep.streamk) &&
      grid > num_sms() * resident_blocks(gemm_tc_kernel<BN, EPI, AR>, GEMM_THREADS, (int)C::SMEM))
    return -1;
  // FRAG_GEMM_TRACE=<file>: tooling only (tools/gemm_trace.py) -- per-CTA
  // globaltimer stamps [start, after PDL wait, first stage, last MMA,
  // accumulator ready, partial written, end] appended after the launch
  static const char* trace_path = std::getenv("FRAG_GEMM_TRACE");
  static unsigned long long* trace_dev = nullptr;
  EpiParams et = ep;
  if (!et.fault) et.fault = fault_slot_current();
  et.spin_ns = spin_limit_ns();
  if (trace_path) {
    if (!trace_dev) cudaMalloc(&trace_dev, 256 * 8 * sizeof(unsigned long long));
    cudaMemsetAsync(trace_dev, 0, 256 * 8 * sizeof(unsigned long long), stream);
    et.trace = trace_dev;
  }
  launch_pdl(gemm_tc_kernel<BN, EPI, AR>, dim3(grid), dim3(GEMM_THREADS), C::SMEM, stream, ta, tb, M, N, K, et);
  if (trace_path) {
    unsigned long long h[256 * 8];
    cudaMemcpyAsync(h, trace_dev, sizeof(h), cudaMemcpyDeviceToHost, stream);
    cudaStreamSynchronize(stream);
    if (FILE* f = std::fopen(trace_path, "ab")) {
      std::fwrite(h, sizeof(h), 1, f);
      std::fclose(f);
    }
  }
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

template <int BN, int AR = BM>
int dispatch_epi(const bf16* A, const bf16* B, int M, int N, int K, EpiKind epi, const EpiParams& ep,
                 cudaStream_t s) {
  switch (epi) {
    case EPI_STORE_BF16: return launch<BN, EPI_STORE_BF16, AR>(A, B, M, N, K, ep, s);
    case EPI_STORE_F32: return launch<BN, EPI_STORE_F32, AR>(A, B, M, N, K, ep, s);
    case EPI_RESID: return launch<BN, EPI_RESID, AR>(A, B, M, N, K, ep, s);
    case EPI_SWIGLU: return launch<BN, EPI_SWIGLU, AR>(A, B, M, N, K, ep, s);
    case EPI_QKV: return launch<BN, EPI_QKV, AR>(A, B, M, N, K, ep, s);
  }
  return -1;
}

}  // namespace

bool smem_attr_needed(const void* fn, int dev) {
  static std::mutex mu;
  static std::unordered_map<const void*, unsigned long long> done;
  std::lock_guard<std::mutex> g(mu);
  unsigned long long& m = done[fn];
  const unsigned long long bit = 1ull << (dev & 63);
  if (m & bit) return false;
  m |= bit;
  return true;
}

int resident_blocks_cached(const void* fn, int dev, int threads, int smem, int (*calc)(const void*, int, int)) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int, int>, int> done;
  std::lock_guard<std::mutex> g(mu);
  const auto key = std::make_tuple(fn, dev, threads, smem);
  auto it = done.find(key);
  if (it != done.end()) return it->second;
  const int n = calc(fn, threads, smem);
  done[key] = n;
  return n;
}

int num_sms() {
  static std::atomic<int> cache[kMaxDevices];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) dev = 0;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (n == 0) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

namespace {
std::atomic<unsigned long long> g_spin_ns{0};
int* g_fault_host = nullptr;  // kMaxDevices ints, mapped + portable pinned memory
std::mutex g_fault_mu;
}  // namespace

unsigned long long spin_limit_ns() {
  unsigned long long v = g_spin_ns.load(std::memory_order_relaxed);
  if (v == 0) {
    const char* e = std::getenv("FRAG_SPIN_LIMIT_MS");
    const double ms = e ? std::atof(e) : 2000.0;
    v = ms > 0 ? (unsigned long long)(ms * 1e6) : 2000000000ull;
    g_spin_ns.store(v, std::memory_order_relaxed);
  }
  return v;
}

void set_spin_limit_ns(unsigned long long ns) { g_spin_ns.store(ns, std::memory_order_relaxed); }

int* fault_slot(int dev) {
  if (dev < 0 || dev >= kMaxDevices) return nullptr;
  std::lock_guard<std::mutex> g(g_fault_mu);
  if (!g_fault_host) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, kMaxDevices * 32 * sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess)
      return nullptr;
    std::memset(p, 0, kMaxDevices * 32 * sizeof(int));
    g_fault_host = static_cast<int*>(p);
  }
  int* h = g_fault_host + dev * 32;  // one 128-byte line per device
  void* d = nullptr;
  if (cudaHostGetDevicePointer(&d, h, 0) != cudaSuccess) return nullptr;
  return static_cast<int*>(d);
}

int* fault_slot_current() {
  int dev = 0;
  cudaGetDevice(&dev);
  static thread_local int last_dev = -1;
  static thread_local int* last_slot = nullptr;
  if (dev != last_dev || !last_slot) {
    last_slot = fault_slot(dev);
    last_dev = dev;
  }
  return last_slot;
}

bool fault_take(int dev) {
  if (dev < 0 || dev >= kMaxDevices) return false;
  {
    std::lock_guard<std::mutex> g(g_fault_mu);
    if (!g_fault_host) return false;
  }
  volatile int* h = g_fault_host + dev * 32;
  if (*h == 0) return false;
  *h = 0;
  return true;
}

// Pick the N tile: maximise useful MMA work per wave while keeping tiles wide
// enough to stay under the shared-memory bandwidth bound (BN=256 moves 96 B/clk
// per SM at full MMA rate, BN=128 128 B/clk, BN=64 192 B/clk).
namespace {
// Tail split for the last partial wave: S K-ranges per leftover tile so the
// leftover tiles occupy (about) one full wave of SMs.
int tail_splits(long tiles, long sms, long nk) {
  const long rem = tiles % sms;
  if (rem == 0) return 1;
  long s = sms / rem;
  if (s > 8) s = 8;
  while (s > 1 && nk / s < 4) --s;
  return (int)(s < 1 ? 1 : s);
}
}  // namespace

// Pick the N tile. Policy measured on B200 with tools/gemm_tune.py
// (profiles/gemm_tune_r01.txt): weight-streaming small-M GEMMs want many CTAs
// (BN=64, BN=128 for very wide N); at M~2.5k BN=128 wins for the N=4k/6k
// projections and BN=256 for the wide gate/up; long-K (down projection) wants
// BN=128 with the tail wave split along K; large M (full prefill) wants BN=256.
// Long-K split-K (the FFN down projection, K = 14336: 224 k-blocks) takes
// strided k-blocks: its A operand (the SwiGLU activations) is produced by the
// gate/up op in two partial waves, and in the GEMM chain a contiguous split
// whose k-range maps onto the second wave could only start after it; strided,
// every split holds the same share of late columns and finishes right behind
// gate/up. Same rule in the chain and here (bit-identical). FRAG_KSTRIDE=0: off.
bool k_strided_for(long nk) {
  static const bool on = [] {
    const char* v = std::getenv("FRAG_KSTRIDE");
    return !(v && v[0] == '0');
  }();
  return on && nk >= 128;
}

static bool pair224_on() {  // FRAG_GEMM_BN224=0: candidates 256 / 192 only
  static const bool on = [] {
    const char* v = std::getenv("FRAG_GEMM_BN224");
    return !(v && v[0] == '0');
  }();
  return on;
}

int gemm_pick_bn(int M, int N, int K) {
  const int m_tiles = (M + BM - 1) / BM;
  int bn;
  if (M <= BM) bn = N >= 16384 ? 128 : 64;
  else if (m_tiles >= 64) bn = 256;
  else if (K >= 8192) bn = 128;
  else if (N >= 16384) bn = 256;
  else bn = 128;
  while (bn > 64 && N % bn) bn >>= 1;
  return bn;
}

int gemm_bf16_tc(const bf16* A, const bf16* B, int M, int N, int K, EpiKind epi, const EpiParams& ep0,
                 cudaStream_t stream, int force_bn_flags) {
  // force_bn_flags: 0 = automatic; else BN in the low 16 bits (64/128/256),
  // bit 16 = still allow the tail split-K, bit 17 = forbid it (tuning only)
  const int force_bn = force_bn_flags & 0xffff;
  if (force_bn_flags & 0x40000)
    return gemm_bf16_tc_pair(A, B, M, N, K, epi, ep0, stream, force_bn ? force_bn : 256,
                             (force_bn_flags & 0x10000) != 0);
  const bool tail_ok = force_bn ? (force_bn_flags & 0x10000) != 0 : (force_bn_flags & 0x20000) == 0;
  if (M <= 0) return 0;
  if (K % BK != 0 || N % 64 != 0) return -1;
  EpiParams ep = ep0;
  ep.splits = 1;
  int bn = force_bn ? force_bn : gemm_pick_bn(M, N, K);
  const int force_splits = (force_bn_flags >> 20) & 0xf;  // tuning: fixed small-M split count
  if (M <= BM && ep.ws && ep.counters) {
    // One M tile (question pass, lm_head rows): a pure weight stream. BN=128
    // and deterministic split-K up to one full wave of CTAs (a second partial
    // round or a fixup per extra split costs more than it saves; measured with
    // tools/gemm_small.py, profiles/gemm_small_r01.txt).
    if (!force_bn) bn = N % 128 == 0 ? 128 : 64;
    const long tiles = N / bn, sms = (long)num_sms(), nk = K / BK;
    long s = 1;
    while (s < 8 && tiles * (s + 1) <= sms && nk / (s + 1) >= 4) ++s;
    if (force_splits > 0) s = force_splits;
    if (s > nk) s = nk;  // every split needs at least one K block
    if (tiles > ep.counters_cap || (size_t)(tiles * s * M * bn) * sizeof(float) > ep.ws_bytes) s = 1;
    ep.splits = (int)s;
    ep.k_strided = s > 1 && k_strided_for(nk) ? 1 : 0;
    ep.full_tiles = 0;
  }
  if (N % bn != 0) return -1;
  const bool want_sk = (force_bn_flags & 0x2000000) != 0;  // tuning: force stream-K
  if (M <= BM && want_sk && ep.ws && ep.counters) {
    // stream-K over the flattened (N tile, k-block) space: every SM streams the
    // same number of weight k-blocks whatever the tile count
    const long long tiles = N / bn, nk = K / BK, I = tiles * nk;
    long long G = num_sms();
    if (I / G < 4) G = I / 4 > 0 ? I / 4 : 1;
    const long long q = I / G;
    const long long maxc = (nk + q - 1) / q + 1;
    if (tiles <= ep.counters_cap && (size_t)(tiles * maxc * M * bn) * sizeof(float) <= ep.ws_bytes) {
      ep.splits = 1;
      ep.streamk = (int)G;
      ep.sk_maxc = (int)maxc;
    }
  }
  // Large M: CTA-pair tiles (256 x 256, cta_group::2) beat every 1-CTA shape in
  // the B200 sweep (profiles/gemm_tune_r01.txt) for the projection shapes.
  if (!force_bn && M >= 256 && N % 256 == 0 && ep.splits == 1) {
    // Wave quantisation on 74 CTA pairs: 192-wide tiles (partial last N tile)
    // when they cut the wave-weighted tile width by >= 5 % (O and down
    // projections at M~2.5k: 160 -> 220 tiles, 3 waves of 0.75 the work; QKV:
    // 4 waves x 256 -> 5 x 192, 109.8 -> 103.9 us in the round-2 ncu sweep,
    // tools/gemm_bn_sweep.sh); otherwise 256 (gate/up, every M~16k shape). Tail split-K only pays for long K (the FFN down
    // projection): at K=4096 the partial write + fixup cost what the shorter
    // last wave saves (tools/gemm_tune.py, profiles/gemm_tune_r01.txt).
    // 224-wide tiles (not SWIGLU, whose gate/up pairs are 64-aligned) join
    // the candidates: QKV at M~2.5k, 4 waves x 224 vs 5 x 192.
    const long m_t = (M + 255) / 256, pairs = num_sms() / 2;
    auto width = [&](long bn) { return (m_t * ((N + bn - 1) / bn) + pairs - 1) / pairs * bn; };
    const long w256 = width(256);
    int bn2 = 256;
    long best = w256;
    for (int cand : {224, 192}) {
      if (cand == 224 && (epi == EPI_SWIGLU || !pair224_on())) continue;
      const long w = width(cand);
      if (w * 100 <= w256 * 95 && w < best) best = w, bn2 = cand;
    }
    return gemm_bf16_tc_pair(A, B, M, N, K, epi, ep, stream, bn2,
                             (force_bn_flags & 0x20000) == 0 && K >= 8192);
  }
  if (ep.splits == 1 && tail_ok && M > BM && (M + BM - 1) / BM < 64 && K >= 8192 && ep.ws && ep.counters) {
    // split-K only the last partial wave (deterministic last-CTA reduction)
    const long tiles = (long)((M + BM - 1) / BM) * (N / bn), sms = num_sms();
    const int s = tail_splits(tiles, sms, K / BK);
    const long tail = tiles % sms;
    if (s > 1 && tail <= ep.counters_cap &&
        (size_t)tail * s * BM * bn * sizeof(float) <= ep.ws_bytes) {
      ep.splits = s;
      ep.full_tiles = (int)(tiles - tail);
    }
  }
  // one-M-tile weight streaming at BN=128: load only the live A rows (32 / 64)
  // per stage -> 20-24 KB stages, 7-8 of them (bit 27 of the flags: force the
  // full 128-row A box, tuning only)
  if (bn == 128 && M <= 64 && !(force_bn_flags & 0x8000000)) {
    if (M <= 32) return dispatch_epi<128, 32>(A, B, M, N, K, epi, ep, stream);
    return dispatch_epi<128, 64>(A, B, M, N, K, epi, ep, stream);
  }
  switch (bn) {
    case 256: return dispatch_epi<256>(A, B, M, N, K, epi, ep, stream);
    case 128: return dispatch_epi<128>(A, B, M, N, K, epi, ep, stream);
    case 64: return dispatch_epi<64>(A, B, M, N, K, epi, ep, stream);
  }
  return -1;
}

}  // namespace fragk
