// Internal host-side objects behind the C ABI: the engine (weights, RoPE
// tables, system-prompt KV cache), the HBM chunk-KV store and the per-request
// result (fused cache + workspace). Host C++ orchestrates; every device step
// is one of the kernels declared in kernels.h.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <shared_mutex>
#include <tuple>
#include <string>
#include <unordered_map>
#include <vector>

#include "frag/frag_c.h"
#include "kernels.h"

namespace fragimpl {

using fragk::bf16;

// ---------------------------------------------------------------- errors
struct Error {
  frag_status code;
  std::string msg;
  int format_kind = -1;  // FRAG_FORMAT_* for FRAG_E_FORMAT
};
[[noreturn]] void fail(frag_status code, const std::string& msg);
[[noreturn]] void fail_format(int kind, const std::string& msg);
void check_cuda(cudaError_t e, const char* what);
void set_last_error(const std::string& m);

extern std::atomic<uint64_t> g_launches;
extern std::atomic<uint64_t> g_alloc_epoch;  // bumped on every device (re)allocation

// Device memory helper (RAII).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  void alloc(size_t n);        // exact allocation (fails with FRAG_E_OOM)
  void ensure(size_t n);       // grow-only
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

struct PinnedBuf {
  void* p = nullptr;
  size_t bytes = 0;
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
  void ensure(size_t n);
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev);
  ~DeviceGuard();
};

// ---------------------------------------------------------------- profiling
// KC_GEMM: tensor-bound GEMMs (M > 128 rows); KC_GEMM_STREAM: one-M-tile
// GEMMs (question pass, lm_head rows), bound by the weight stream from HBM.
// KC_GEMM_GU: the gate/up projection at M > 128 alone (also counted in KC_GEMM)
// KC_VWIN: shared V pages, the per-layer V window fills of the large passes
enum KClass { KC_GEMM = 0, KC_ATTN = 1, KC_STITCH = 2, KC_NORM = 3, KC_SELECT = 4, KC_GEMM_STREAM = 5, KC_GEMM_GU = 6,
              KC_VWIN = 7, KC_N = 8 };
inline int gemm_class(int M) { return M <= 128 ? KC_GEMM_STREAM : KC_GEMM; }
struct Profiler {
  bool on = false;
  struct Rec {
    cudaEvent_t a, b;
    int klass;
    double flops, bytes;
    int launches;
  };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> pool;
  double ms[KC_N] = {}, flops[KC_N] = {}, bytes[KC_N] = {};
  int64_t launches[KC_N] = {};
  std::mutex mu;
  cudaEvent_t get();
  void begin(cudaStream_t s, cudaEvent_t* a);
  void end(cudaStream_t s, cudaEvent_t a, int klass, double flops, double bytes, int launches);
  void collect();  // after the stream is synchronised
  void reset();
  ~Profiler();
};

// ---------------------------------------------------------------- store
struct ChunkKey {
  uint64_t a, b;
  bool operator==(const ChunkKey& o) const { return a == o.a && b == o.b; }
};
struct ChunkKeyHash {
  size_t operator()(const ChunkKey& k) const { return (size_t)(k.a ^ (k.b * 0x9e3779b97f4a7c15ULL)); }
};
ChunkKey key_of(const frag_chunk_id& id);

// Shared ownership: a result whose V rows are read in place from a record
// (shared V pages) keeps the record's pages alive until its next request.
struct Record : std::enable_shared_from_this<Record> {
  frag_chunk_id id{};
  int n_tok = 0;
  int native_start = 1;
  int variant = FRAG_VARIANT_ISOLATED;
  uint64_t heat = 0, last_access = 0;
  int pins = 0;
  size_t bytes = 0;
  DevBuf kv;            // K then V, each [L][n][Hkv][dh] bf16
  DevBuf tok;           // int32 [n]
  std::vector<int32_t> tok_host;
  // chunk-partitioned store: an imported record is a view of
  // another process's record pages mapped through CUDA IPC (read over NVLink
  // by K1); the mapping is closed, never freed, when the view is dropped
  int tier = FRAG_TIER_GPU;
  int owner_device = -1;
  bool ipc_mapped = false;
  bool exported = false;  // IPC handle handed out: never replaced while peers may map it
  bf16* k() const { return kv.as<bf16>(); }
  bf16* v() const { return kv.as<bf16>() + kv.bytes / 4; }
  Record() = default;
  Record(const Record&) = delete;
  Record& operator=(const Record&) = delete;
  ~Record();
};

struct Store {
  frag_model_cfg cfg{};
  int device = 0;
  size_t capacity = 0, used = 0;
  uint64_t tick = 0;
  mutable std::shared_mutex mu;
  std::unordered_map<ChunkKey, std::shared_ptr<Record>, ChunkKeyHash> recs;
  // same-process stores on other GPUs whose records this store serves on a
  // local miss (frag_store_attach_peer); their pages are read over NVLink
  std::vector<Store*> peers;
  // alternative_path_match prefix index: PrefixKey(sys, path) -> last chunk of the path
  std::unordered_map<ChunkKey, ChunkKey, ChunkKeyHash> prefix_index;
  size_t record_bytes(int n_tok) const {
    return (size_t)2 * cfg.layers * n_tok * cfg.n_kv_heads * cfg.head_dim * sizeof(bf16);
  }
};

// ---------------------------------------------------------------- engine
struct LayerW {
  bf16 *wqkv, *wo, *wgu, *wd, *attn_norm, *ffn_norm;
};

struct SysKV {
  int n = 0;
  DevBuf kv;  // K then V [L][n][Hkv][dh]
};

struct Result;

struct Engine {
  frag_model_cfg cfg{};
  int device = 0;
  uint64_t seed = 0;
  DevBuf weights;  // one allocation for every tensor
  bf16 *emb = nullptr, *lm_head = nullptr, *final_norm = nullptr;
  std::vector<LayerW> layers;
  size_t n_params = 0;
  // RoPE table [rows][dh/2] (cos, sin) of (row+1)*theta_i computed in fp64
  DevBuf rope;
  int rope_rows = 0;
  std::vector<double> theta;  // theta_i, i = 1..dh/2
  std::mutex rope_mu;         // guards rope-table growth
  std::mutex mu;              // guards the system-prompt cache and the scratch result
  std::map<std::vector<int32_t>, std::unique_ptr<SysKV>> sys_cache;
  Profiler prof;
  std::unique_ptr<Result> scratch;  // preprocess / system-prompt prefill workspace

  void ensure_rope(int rows);
  size_t qkv_cols() const { return (size_t)(cfg.n_heads + 2 * cfg.n_kv_heads) * cfg.head_dim; }
};

// Serialises the device work of every engine's calls on one device, process
// wide: the persistent GEMMs (split-K fixups, stream-K owners, the GEMM chain)
// spin on other CTAs of their own grid and assume it is co-resident, i.e. owns
// the GPU while it runs. Every call synchronises before it returns, so holding
// this for the call suffices inside one process; across processes the bounded
// waits (ptx.cuh spin_until_ge) turn a missing co-residency into FRAG_E_CUDA.
std::recursive_mutex& device_mutex(int device);

// Shape of a request body; a captured CUDA graph is valid for one key.
struct GraphKey {
  int T, S, N, nq, k, inject, all_logits, raw, logits_on_device, n_desc, max_rows, selector;
  uint64_t rope;
  std::vector<int> shapes = {};  // batched reprocess: per-request (T, S, N, |Q|, k), exact
  bool operator<(const GraphKey& o) const {
    return std::tie(T, S, N, nq, k, inject, all_logits, raw, logits_on_device, n_desc, max_rows, selector, rope,
                    shapes) <
           std::tie(o.T, o.S, o.N, o.nq, o.k, o.inject, o.all_logits, o.raw, o.logits_on_device, o.n_desc,
                    o.max_rows, o.selector, o.rope, o.shapes);
  }
};
struct GraphEntry {
  cudaGraphExec_t exec = nullptr;
  uint64_t epoch = 0;
  uint64_t launches = 0;
};
struct StitchPlan {
  int n_desc = 0, max_rows = 0;
  double bytes = 0;
};

struct Result {
  Engine* eng = nullptr;
  std::map<GraphKey, GraphEntry> graphs;
  std::set<GraphKey> seen;
  cudaStream_t cap_stream = nullptr;
  // K1 per layer on a side stream overlapping the question pass
  cudaStream_t side = nullptr;
  cudaEvent_t fork_ev = nullptr;
  std::vector<cudaEvent_t> layer_ev;
  // shared V window fills on the side stream: [0, L) attention of layer l done
  // (its window buffer is free), [L, 2L) window of layer l filled
  std::vector<cudaEvent_t> vwin_ev;
  int max_tokens = 0;
  // fused cache [L][max_tokens][Hkv][dh]
  DevBuf k_fused, v_fused;
  int T = 0, S = 0, N = 0, nq = 0, k_sel = 0, M = 0, logit_rows = 0;
  // batched requests (reprocess_batch): request b owns cache rows
  // [b * rows_per_seq, ...); 0 = one sequence
  int rows_per_seq = 0;
  struct BatchReq {
    int T, S, N, nq, k, plan_off;
    std::vector<int32_t> crit;  // host copy after the request (1-based positions)
  };
  std::vector<BatchReq> batch;
  // workspace
  DevBuf h, x, q, attn, act, plan_rows, plan_tok, chunk_tok, q_tok, q_final, scores, part_ms, row_ms, part_o,
      part_lse, logits, row_map, stitch_desc, stitch_tab, lm_x, gemm_ws, gemm_cnt, dec_tok, fr_save, dev, score_col, score_q,
      ssq;
  PinnedBuf staging, logits_host;
  // shared V pages: with vshared the V
  // rows of the chunks (and KV_S) are read in place from their records through
  // the per-sequence patch plans; only this request's fresh rows live in vx
  // (exclusive slots: critical rows at their GEMM row, question / decoded rows
  // by rule). v_fused then exists only as the read-back view.
  bool vshared = false;
  bool v_materialized = false;  // v_fused holds the view of the current request
  int vx_rows = 0;              // exclusive slots per layer
  int v_tail_row0 = 0x7fffffff, v_tail_slot0 = 0;  // QKV epilogue slot rule (one sequence)
  struct VSeq {
    int seg0, n_seg;         // segments in vseg
    int vt_off, vp_off, ve_off, n_rows;  // plan slices (vplan_tile / vplan_prim / vplan_ent)
    int base, T;             // cache rows of the sequence
    int tail_row0;           // sequence-local first question row
    int tail_slot_q, tail_slot_s;  // exclusive slot of that row in the question / sparse pass
  };
  std::vector<VSeq> vseq;
  DevBuf vx, vx_map, vseg, vplan_args, vplan_tile, vplan_prim, vplan_ent;
  DevBuf vwin;  // large passes: V of one layer staged at its cache rows, double-buffered [2][max_tokens]
  int vseg_n = 0, vseg_max_rows = 0, vseg_rows = 0;
  std::vector<std::shared_ptr<Record>> vrefs;  // records whose pages the shared V view reads
  bool q_final_in_full = false;  // PASS_FULL also keeps the last layer's fp32 queries (r = 0 fast path)
  // timing
  cudaEvent_t ev[7] = {};
  bool timing_valid = false;
  frag_timing timing{};
  cudaStream_t last_stream = nullptr;
  bool logits_on_device = false;
  ~Result();
};

Engine* engine_create(const frag_model_cfg& cfg, int device, uint64_t seed);
void result_init(Result* r, Engine* e, int max_tokens);
// The request about to run keeps a private fused V [L][max_tokens] (full
// prefill, CacheBlend, peer records, scratch passes) instead of shared pages.
void use_private_v(Result* r);
// Shared V pages: write the fused V view of the current request into v_fused
// (frag_result_fused_kv read-back); a no-op for a private V.
void materialize_v(Result* r, cudaStream_t s);
int set_shared_v(int on);  // 1 / 0 sets, -1 queries; returns the previous setting
uint64_t result_device_bytes(const Result* r);

// Pipeline stages (engine.cpp)
enum PassMode { PASS_FULL = 0, PASS_QUESTION = 1, PASS_KV_ONLY = 2 };
// Run every layer over the M planned rows (plan_rows/plan_tok on device) of the
// result's fused cache with T valid rows; PASS_QUESTION stops after the final
// layer's QKV projection with fp32 queries in r->q_final; PASS_FULL ends with
// logits for the rows listed in row_map (n_logit_rows of them, device).
// n_layers > 0 runs only the first n_layers layers (a non-FULL pass then stops
// after layer n_layers-1's QKV projection: kv_deviation's 2-layer FA pass).
// layer_ready: optional per-layer events the stream waits on before layer l's
// attention (the stitch of that layer running on another stream).
// segs: optional batched sequences (plan-row ranges over their own cache slices)
struct Seg {
  int off;      // first plan row of the sequence
  int M;        // plan rows of the sequence
  int base;     // first fused-cache row of the sequence
  int T;        // cache rows visible to the sequence
  int seq = 0;  // sequence index (shared V pages: Result::vseq)
};
void run_rows(Engine* e, Result* r, cudaStream_t s, int M, int T, PassMode mode, const int* row_map_dev,
              int n_logit_rows, int n_layers = 0, const cudaEvent_t* layer_ready = nullptr,
              const std::vector<Seg>* segs = nullptr, int keep_last = 0);
// keep_last > 0 (PASS_FULL, one sequence): only the trailing keep_last rows'
// final-layer hidden states are needed (the logit rows), so the last layer
// runs attention / O / MLP on those rows only (all rows' K/V still written).

void reprocess(Engine* e, Store* st, const int32_t* sys, int n_sys, const int32_t* q_tokens, int n_q,
               bool q_on_device, const frag_chunk_id* ids, int n_chunks, float ratio, const frag_reprocess_opts* o,
               cudaStream_t s, Result* r);
void full_prefill(Engine* e, const int32_t* sys, int n_sys, const int32_t* tokens, int n_tok,
                  const frag_reprocess_opts* o, cudaStream_t s, Result* r);
void reprocess_batch(Engine* e, Store* st, const frag_request* reqs, int B, int slot, const frag_reprocess_opts* o,
                     cudaStream_t s, Result* r);
// kv_deviation (Eq. 7): Full Reuse (stitched) vs Full Attention
// over cat(S, chunks) through the first n_layers layers; dev_host [N][n_layers][2]
// (K, V). The result holds the Full-Reuse stitched cache afterwards.
void kv_deviation(Engine* e, Store* st, const int32_t* sys, int n_sys, const frag_chunk_id* ids, int n_chunks,
                  int n_layers, cudaStream_t s, Result* r, float* dev_host);
// Greedy decoding after a reprocess / full prefill: token 0 =
// argmax of the last logits row, then n_new-1 single-row steps at positions
// T+1.. whose K/V are appended to the result's own fused cache (its exclusive
// pages); the shared records are never touched.
void decode(Engine* e, Result* r, int n_new, cudaStream_t s, int32_t* out_host);
void preprocess_isolated(Engine* e, Store* st, const int32_t* sys, int n_sys, const int32_t* tokens, int n_tok,
                         bool overwrite, frag_chunk_id* id_out);
void preprocess_fused(Engine* e, Store* src, Store* dst, const int32_t* sys, int n_sys, const int32_t* tokens,
                      int n_tok, const frag_chunk_id* nb, int n_nb, int budget, bool overwrite, frag_chunk_id* id_out);

// Store operations (store.cpp)
Store* store_create(const frag_model_cfg& cfg, int device, size_t cap);
void store_put(Store* st, const frag_chunk_id& id, const int32_t* tokens, int n_tok, int native_start, int variant,
               const void* k, const void* v, bool overwrite, size_t src_layer_pitch_elems = 0,
               cudaStream_t s = nullptr);
Record* store_fetch(Store* st, const frag_chunk_id& id);      // heat++, pin; StoreError when missing
Record* store_try_fetch(Store* st, const frag_chunk_id& id);  // same, nullptr when missing
// FKVC record files (serialize_record / deserialize_record): fp32
// K then V per layer; tokens are supplied by the caller (the format omits them).
void store_save(Store* st, const frag_chunk_id& id, const char* path);
void store_load(Store* st, const char* path, const int32_t* tokens, int n_tok, bool overwrite, cudaStream_t s,
                frag_chunk_id* id_out);
void fkvc_write(const char* path, const frag_fkvc_header& h, const float* k, const float* v);
void fkvc_read(const char* path, frag_fkvc_header* h, float* k, float* v, size_t cap_floats);
void store_release(Store* st, const frag_chunk_id& id);
// FKVC manifest (manifest.cpp): chunk_id -> relative path +
// variant + native_start (+ the chunk's token ids)
struct ManifestEntry {
  frag_chunk_id id{};
  std::string path;  // resolved against the manifest's directory
  int variant = FRAG_VARIANT_ISOLATED;
  int32_t native_start = 1;
  std::vector<int32_t> tokens;
};
std::vector<ManifestEntry> manifest_read(const char* path);  // host only; checks every file header
int manifest_save(Store* st, const char* dir, const char* name);
int manifest_load(Store* st, const char* path, bool overwrite, cudaStream_t s);
// chunk-partitioned store across GPUs: same-process peers and
// cross-process CUDA-IPC export/import of record pages
int32_t chunk_owner(const frag_chunk_id& id, int32_t n);
void store_attach_peer(Store* local, Store* remote);
ChunkKey prefix_key(const frag_chunk_id* sys_id, const frag_chunk_id* path, int n);
void store_register_prefix(Store* st, const frag_chunk_id* sys_id, const frag_chunk_id* path, int n);
int store_match(Store* st, const frag_chunk_id* sys_id, const frag_chunk_id* ctx, int n, frag_match* out);
void store_export(Store* st, const frag_chunk_id& id, frag_peer_record* out);
void store_import(Store* st, const frag_peer_record& pr, const int32_t* tokens, int n_tok, bool overwrite);

void hash_tokens(const int32_t* t, int n, uint64_t salt, frag_chunk_id* out);
uint64_t weight_seed(uint64_t seed, int tensor_id);

}  // namespace fragimpl
