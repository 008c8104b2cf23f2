// Host-side launchers for the sm_100a kernels of the reprocessing path.
// Every pointer is a device pointer; every launcher is stream-ordered and
// never synchronises. Kernel numbering (K1..K11) follows SURVEY.md §2.2.
#pragma once
#include <cstddef>
#include <utility>
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace fragk {

using bf16 = __nv_bfloat16;

// ------------------------------------------------------------------ GEMM
// C[M,N] = A[M,K] · B[N,K]^T, A/B bf16 K-major, fp32 accumulation in TMEM.
enum EpiKind : int {
  EPI_STORE_BF16 = 0,  // out_bf16[row*ldo + col] = acc
  EPI_STORE_F32 = 1,   // out_f32[row*ldo + col] = acc
  EPI_RESID = 2,       // resid[row*ldo + col] += acc            (K7, K8-down)
  EPI_SWIGLU = 3,      // 32-col gate/up interleave -> out_bf16[row*ldo + j] = silu(g)*u   (K8-gate/up)
  EPI_QKV = 4,         // RoPE(Q,K) at rows[row]; Q -> q_out, K/V scattered into the fused cache (K4+K5)
};

struct EpiParams {
  int ldo = 0;
  float* out_f32 = nullptr;
  bf16* out_bf16 = nullptr;
  float* resid = nullptr;
  // EPI_QKV
  const int* rows = nullptr;       // fused-cache row (position-1) of each GEMM row
  const float2* rope = nullptr;    // [pos_row][dh/2] (cos, sin) of (row+1)*theta_i
  int rows_per_seq = 0;            // > 0: position row = row % rows_per_seq (batched sequences)
  bf16* q_out = nullptr;           // [M][Hq][dh]
  float* q_out_f32 = nullptr;      // optional fp32 copy (question pass, final layer)
  bf16* k_cache = nullptr;         // layer base, [T][Hkv][dh]
  bf16* v_cache = nullptr;         // layer base: [T] rows, or the exclusive slots (v_slots)
  // shared V pages: fresh V goes to exclusive slot = row (GEMM row), or for a
  // position row >= v_tail_row0: v_tail_slot0 + prow - v_tail_row0
  int v_slots = 0;
  int v_tail_row0 = 0x7fffffff, v_tail_slot0 = 0;
  bf16* v_cache2 = nullptr;        // shared V pages, staged window of this layer: fresh V also at [prow]
  int Hq = 0, Hkv = 0, dh = 0;
  // split-K workspace for small-M GEMMs (owned by the caller's result; the
  // counters must start at zero and are left at zero by the kernel)
  float* ws = nullptr;
  size_t ws_bytes = 0;
  int* counters = nullptr;
  int counters_cap = 0;
  int splits = 1;      // set by gemm_bf16_tc: K splits of each tail tile
  int full_tiles = 0;  // tiles before the split tail
  int streamk = 0;     // set by gemm_bf16_tc: stream-K decomposition (one M tile)
  int k_strided = 0;   // one-M-tile split-K: split sp takes k-blocks sp, sp+S, ... (long K, see gemm_tc.cu)
  int group_m = 0;     // CTA-pair GEMM tile raster: M blocks per group (0: all, M fastest)
  int sk_maxc = 0;     // stream-K: max CTAs sharing one tile (workspace slots per tile)
  unsigned long long* trace = nullptr;  // tooling: per-CTA globaltimer stamps (FRAG_GEMM_TRACE)
  // RMSNorm folded into the GEMMs (K3): norm(h)·Wᵀ = rs(h) · (h·Wᵀ) with unit
  // gains, rs = rsqrt(mean(h²) + eps). The EPI_RESID epilogue that updates h
  // also writes bf16(h) (the next GEMM's A operand) and one partial Σh² per
  // 32-column chunk; the consuming EPI_QKV / EPI_SWIGLU epilogue sums the
  // partials of its row in chunk order and scales the accumulator by rs.
  float* ssq_out = nullptr;       // EPI_RESID: [d/32][ssq_ld] partial sums of squares
  bf16* x_out = nullptr;          // EPI_RESID: bf16(h), row stride ldo
  const float* ssq_in = nullptr;  // EPI_QKV / EPI_SWIGLU: the producer's partials
  int ssq_ld = 0;                 // row stride of the partials
  int ssq_n = 0;                  // partials per row (d/32)
  int norm_d = 0;
  float norm_eps = 0.f;
  // 1 inside the GEMM chain: ops of one launch read data other CTAs wrote
  // earlier in it (residual, Σh² partials), which L1 does not keep coherent --
  // those reads go to L2 (ld.global.cg)
  int l2_reads = 0;
  // bounded inter-CTA waits (ptx.cuh spin_until_ge): the device's mapped host
  // fault slot and the wait limit; filled in by the launchers
  int* fault = nullptr;
  unsigned long long spin_ns = 0;
};

struct GemmTimer;  // optional per-launch event hook (bench roofline)

// Returns the number of kernel launches issued (1), or -1 on a shape error.
int gemm_bf16_tc(const bf16* A, const bf16* B, int M, int N, int K, EpiKind epi, const EpiParams& ep,
                 cudaStream_t stream, int force_bn = 0);
int gemm_pick_bn(int M, int N, int K);
// CTA-pair (cta_group::2) variant: 256 x bn tiles (bn = 128 or 256); the last
// partial wave split along K unless tail_split is false.
int gemm_bf16_tc_pair(const bf16* A, const bf16* B, int M, int N, int K, EpiKind epi, const EpiParams& ep,
                      cudaStream_t stream, int bn, bool tail_split = true);
int num_sms();  // SM count of the current device (cached per device)
// Co-residency fault slot of `dev` (mapped pinned host memory, device-visible)
// and the inter-CTA wait limit (FRAG_SPIN_LIMIT_MS, default 2000 ms).
int* fault_slot(int dev);
int* fault_slot_current();
unsigned long long spin_limit_ns();
void set_spin_limit_ns(unsigned long long ns);  // tests / tooling
// Reads and clears the slot after the stream has been synchronised: true if a
// persistent grid abandoned an inter-CTA wait since the last call.
bool fault_take(int dev);

// Weight-streaming GEMM chain (gemm_chain.cu): up to CHAIN_MAX_OPS one-M-tile
// GEMMs (M <= 128 rows, BN = 128) in one persistent launch, op i+1's A = op i's
// output. `done` = 2*CHAIN_MAX_OPS ints, zero before the first launch (left zero).
constexpr int CHAIN_MAX_OPS = 4;
bool k_strided_for(long nk);  // one-M-tile split-K over strided k-blocks (gemm_tc.cu)
struct AttnArgs;
struct ChainStep {
  const bf16* A = nullptr;
  const bf16* B = nullptr;
  int N = 0, K = 0;
  EpiKind epi = EPI_STORE_BF16;
  EpiParams ep;
};
struct ChainOp {
  int N, K, epi, splits;
  int sp_major;  // split units numbered split-major (all tiles' split 0 first)
  EpiParams ep;
};
bool gemm_chain_supported(int M, int N, int K);
// pre_combine: split-KV attention whose combine (-> op 0's A operand) runs
// inside the chain before op 0 (nullptr: none)
int gemm_chain_tc(const ChainStep* steps, int n_ops, int M, int* done, cudaStream_t stream,
                  const AttnArgs* pre_combine = nullptr);

// TMA descriptors (bf16, SWIZZLE_128B, 64-element inner box), encoded through the
// driver entry point so the library needs no link-time libcuda.
bool make_tmap_2d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t row_stride_elems,
                  uint32_t box_rows);
bool make_tmap_3d(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1_elems,
                  uint64_t s2_elems, uint32_t b0, uint32_t b1, uint32_t b2);

// ------------------------------------------------------------------ K1
struct StitchChunk {
  const bf16* k_src;   // record K [L][n][Hkv][dh]
  const bf16* v_src;   // record V
  int n_tok;           // rows in the record
  int dst_row;         // first fused-cache row (target_start - 1)
  int table;           // index into the per-chunk cos/sin table; -1 = zero shift (bit copy)
};
// fused K/V [L][T][Hkv][dh]; tables: [n_tables][dh/2] float2 for delta*theta_i.
int rope_shift_assemble(const StitchChunk* chunks_dev, int n_chunks, int max_rows, const float2* tables,
                         bf16* k_fused, bf16* v_fused, int L, int T, int Hkv, int dh, cudaStream_t stream,
                         int layer0 = 0);

// ------------------------------------------------------------------ K2/K3
// h[i] = E[tok[i]] (fp32), x[i] = bf16(rmsnorm(h[i]) * g)
void embed_rmsnorm(const bf16* E, const int* tok, int M, int d, const bf16* gain, float eps, float* h, bf16* x,
                   cudaStream_t stream);
void rmsnorm(const float* h, int M, int d, const bf16* gain, float eps, bf16* x, cudaStream_t stream,
             const int* row_map = nullptr);

// ------------------------------------------------------------------ shared V pages
// A request's V rows are read in place from the store's records (shared
// pages, never copied: SPEC.md:148-150); only the rows
// computed for this request (critical + question + decoded tokens) live in its
// exclusive V region, slot-indexed. One VSeg per statically placed source
// (KV_S, each chunk record), sorted by first cache row (sequence-local).
struct alignas(64) VSeg {
  CUtensorMap tmap;   // V [L][n][Hkv*dh] as (Hkv*dh, n, L), box (64, 128, 1), SW128: a tile's primary box
  CUtensorMap tmap1;  // the same tensor, box (64, 1, 1): one patched row
  const bf16* v;      // V base (layer 0, row 0)
  int row0;           // first sequence-local cache row
  int n;              // rows
  int base;           // first cache row of the sequence (batched requests)
  int pad[11];
};
static_assert(sizeof(VSeg) == 320, "VSeg layout");
// Per-sequence patch plan over 128-row key tiles (sequence-local rows): tile
// j's TMA box comes from its primary segment vprim[j] = (segment, row
// coordinate) -- the segment holding row 128j; none: segment 0 at a row past
// its end, i.e. an all-zero box -- and its entries vent[vtile[j] ..
// vtile[j+1]) are the rows that box does not supply: rows of other segments
// and fresh critical rows, in row order. Rows >= tail_row0 (question rows,
// decoded tokens) are fresh by rule (slot = tail_slot0 + row - tail_row0) and
// never planned. entry = row_in_tile | (seg + 1) << 8 (0: exclusive slot) | src_row << 32
struct VPlanArgs {
  const VSeg* segs;
  int n_seg;
  const int* crit;     // ascending critical rows (n_crit), cache rows = local + row_base
  int n_crit;
  int row_base;
  int crit_slot0;      // exclusive slot of crit[0]
  int tail_row0;       // sequence-local; rows >= tail_row0 are fresh by rule
  int n_rows;          // rows covered (tiles = ceil(n_rows / 128))
  int* vtile;          // [tiles + 1]
  int2* vprim;         // [tiles]
  unsigned long long* vent;  // [n_rows]
};
int vpatch_plan(const VPlanArgs* seqs_dev, int n_seq, int max_rows, int max_segs, cudaStream_t stream);
bool vpatch_plan_fits(int max_rows, int max_segs);  // the one-CTA plan's shared memory (rows up to ~800k)
// Large passes (the sparse pass) stage one layer of V at a time: copy every
// segment's layer-`layer` rows into the window dst [cache rows][Hkv*dh] at
// rows base + row0 + i (fresh rows are written there by the QKV epilogue).
int vwindow_fill(const VSeg* segs, int n_seg, int max_rows, int layer, int kvc, bf16* dst, cudaStream_t stream);
// Materialise V rows [0, n_rows) of every layer into dst [L][ld][Hkv*dh] from
// the segments + exclusive region (result read-back: frag_result_fused_kv)
int vpage_gather(const VSeg* segs, const int* vtile, const int2* vprim, const unsigned long long* vent,
                 const bf16* vx, size_t vx_layer_stride, int tail_row0, int tail_slot0, int n_rows, int L, int kvc,
                 bf16* dst, size_t dst_layer_stride, cudaStream_t stream);

// ------------------------------------------------------------------ K6
struct AttnArgs {
  const bf16* q;         // [M][Hq][dh]
  const bf16* k;         // fused layer base [T][Hkv][dh]
  const bf16* v;
  const int* rows;       // [M] query fused-cache row (ascending); row - row_base indexes k/v
  int row_base = 0;      // first cache row of this sequence (batched requests share one cache)
  bf16* out;             // [M][Hq][dh]
  float* part_o;         // split partials [splits][M][Hq][dh]
  float* part_lse;       // [splits][M][Hq]
  int M, T, Hq, Hkv, dh;
  int split_keys;        // keys per split (multiple of 64); <=0: no split
  int n_splits;
  float scale;           // 1/sqrt(dh)
  unsigned long long* trace = nullptr;  // tooling: clock64 timeline of CTA 0 (FRAG_ATTN_TRACE)
  // shared V pages (vsegs != nullptr; `v` unused): V tiles come from the
  // segments' tensor maps, patched from the plan and the exclusive region
  const VSeg* vsegs = nullptr;
  int n_vseg = 0;
  const int* vtile = nullptr;  // this sequence's plan: entry starts [tiles + 1] (tile 0 = sequence row 0)
  const int2* vprim = nullptr; // [tiles] (primary segment, TMA row coordinate)
  const unsigned long long* vent = nullptr;
  const bf16* vx = nullptr;    // exclusive V of this layer: [slot][Hkv][dh]
  const CUtensorMap* vx_map = nullptr;  // exclusive V [L][slots][Hkv*dh] as (Hkv*dh, slots, L): [0] box (64, 1, 1), [1] box (64, 32, 1)
  int layer = 0;
  int tail_row0 = 0x7fffffff, tail_slot0 = 0;
};
// returns launches; with combine_deferred != nullptr a split-KV launch leaves
// the combine to the caller (*combine_deferred = true)
int sparse_q_attention(const AttnArgs& a, cudaStream_t stream, bool* combine_deferred = nullptr);
int attn_tc_launch(const AttnArgs& a, int G, int n_qblocks, cudaStream_t stream);
int attn_rows_per_cta();
bool attn_shared_v_supported(int dh);  // the attention kernels in use read shared V pages

// ------------------------------------------------------------------ K9/K10
struct ScoreArgs {
  const float* q;      // [nq][Hq][dh] fp32 final-layer queries
  const bf16* k;       // final-layer fused K base [T][Hkv][dh]
  int nq, Hq, Hkv, dh;
  int key_row0;        // first chunk row in the fused cache (= |S|)
  int n_keys;          // N chunk tokens
  float scale;
  float2* part_ms;     // [nblk][nq*Hq] (max, sumexp) scratch
  float2* row_ms;      // [nq*Hq] (max, 1/Z)
  float* scores;       // [n_keys]
  int raw;             // 1 = raw (unnormalised) attention logits summed (SPEC.md:464 flag)
  float* col_part;     // [score_col_part_elems] per (kv head, row tile) column partials (tensor path)
  bf16* q_split;       // [score_q_split_elems] three-term bf16 split of q (tensor path)
};
int qg_score(const ScoreArgs& a, cudaStream_t stream);
// tcgen05 scoring (score_tc.cu): 3-term bf16 split of the fp32 queries
int qg_score_tc(const ScoreArgs& a, cudaStream_t stream);
size_t score_col_part_elems(int nq, int Hq, int Hkv, int n_keys);
size_t score_q_split_elems(int nq, int Hq, int Hkv, int dh);
int score_combine(const ScoreArgs& a, int nblk, cudaStream_t stream);
// crit rows (ascending, = key_row0 + j) of the k largest scores, ties to lower j,
// then the question rows appended. Writes plan_rows[k + nq] and plan_tok.
int topk_plan(const float* scores, int n_keys, int k, int key_row0, const int* chunk_tok, const int* q_tok,
              int nq, int q_row0, int* plan_rows, int* plan_tok, cudaStream_t stream);
// kv_deviation (Eq. 7): per chunk token j and layer l < n_layers,
// dev[j][l][0|1] = sum over Hkv*dh of the squared K|V difference between the
// Full-Attention rows (k_fa/v_fa + l*fa_layer_stride + j*width) and the Full-Reuse
// rows (k_fr/v_fr + l*fr_layer_stride + j*width); sel_scores[j] = the sel_comp
// (0 K, 1 V, 2 K+V) deviation at layer sel_layer (select_cacheblend, Eq. 8).
struct DeviationArgs {
  const bf16 *k_fa, *v_fa, *k_fr, *v_fr;
  size_t fa_layer_stride, fr_layer_stride;  // elements
  int n_rows, n_layers, width;
  float* dev;         // [n_rows][n_layers][2] or null
  float* sel_scores;  // [n_rows] or null
  int sel_layer, sel_comp;
};
int kv_deviation(const DeviationArgs& a, cudaStream_t stream);
// Greedy decoding step: argmax(logits[0..V)) (lowest index on ties) -> out[0],
// or out[*out_idx] with *out_idx incremented when out_idx is set; also stored
// as the next step's plan token, and plan_rows[0] = next_row (next_row < 0:
// incremented on the device).
int greedy_argmax(const float* logits, int V, int* out, int* out_idx, int* plan_tok, int* plan_rows, int next_row,
                  cudaStream_t stream);

// ------------------------------------------------------------------ weights
// Fill dst[i] = bf16(normal_f(sigma)) from the counter form of the splitmix64
// stream `seed` (element e = e-th gaussian of the Box-Muller pair sequence).
// Rows of the canonical [rows][cols] tensor land at dst + map(row)*cols where
// map(row) = (row / blk) * blk_stride + blk_off + row % blk.
void init_normal_bf16(bf16* dst, uint64_t seed, size_t rows, size_t cols, float sigma, int blk, int blk_stride,
                      int blk_off, cudaStream_t stream);
void fill_bf16(bf16* dst, size_t n, float v, cudaStream_t stream);
// fp32 -> bf16 round-to-nearest-even, n % 4 == 0 (FKVC loads)
void f32_to_bf16(const float* src, bf16* dst, size_t n, cudaStream_t stream);

}  // namespace fragk

namespace fragk {
// Launch with programmatic stream serialization (PDL): the kernel may start
// while the previous one drains; it must griddepcontrol.wait before touching
// that kernel's outputs.
template <class... KArgs, class... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Raise a kernel's dynamic shared-memory limit once per device (the attribute is
// per device context; setting it on every launch costs a driver round trip).
// Keyed by the kernel's address (instantiations share a function type).
bool smem_attr_needed(const void* fn, int dev);  // marks (fn, dev) as done
template <class Kernel>
inline void smem_attr_once(Kernel* fn, int bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (!smem_attr_needed(reinterpret_cast<const void*>(fn), dev)) return;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

// Co-residency check for the persistent kernels whose CTAs wait on each other
// (split-K fixups, the GEMM chain): CTAs of `fn` that fit on one SM with this
// block size and shared memory, from the occupancy calculator, cached per
// (kernel, device). A grid larger than blocks x SMs could never be resident
// at once, so the launcher refuses it (FRAG_E_CUDA) instead of launching a
// grid whose waits could only end at the spin limit.
int resident_blocks_cached(const void* fn, int dev, int threads, int smem, int (*calc)(const void*, int, int));
template <class Kernel>
inline int resident_blocks(Kernel* fn, int threads, int smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  return resident_blocks_cached(reinterpret_cast<const void*>(fn), dev, threads, smem,
                                [](const void* f, int t, int b) {
                                  int n = 0;
                                  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, (Kernel*)f, t, (size_t)b) !=
                                      cudaSuccess) {
                                    cudaGetLastError();
                                    return 0;
                                  }
                                  return n;
                                });
}
}  // namespace fragk
