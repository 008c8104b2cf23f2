/* frag_c.h — C ABI of the B200-native FusionRAG online reprocessing path.
 *
 * This is the drop-in boundary for the reference's reprocessing surface
 * (namespace frag, /root/reference/proj/include/frag/common.hpp and the
 * operation contracts of /root/reference/SPEC.md). Each entry point cites the
 * reference interface it replaces. Exceptions never cross this boundary: every
 * function returns a frag_status, and frag_last_error() holds a thread-local
 * message. The C++ wrapper (frag/fusion.hpp) re-throws them as the
 * reference's frag::ContractError / StoreError / FormatError.
 *
 * Threading:
 *   - an engine or store is bound to one CUDA device; use one host thread per GPU;
 *   - engine weights are immutable after create; frag_reprocess is reentrant
 *     given distinct result objects;
 *   - store puts take a writer lock, fetches a reader lock, and records are
 *     pinned while a fetch handle is outstanding.
 * Layouts: K/V of a record and of the fused cache are [L][tokens][Hkv][dh]
 * bf16, post-RoPE. Positions are 1-based
 * (common.hpp:15); fused-cache row r holds position r+1.
 */
#ifndef FRAG_C_H
#define FRAG_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define FRAG_API __attribute__((visibility("default")))
#else
#define FRAG_API
#endif

/* Error taxonomy of common.hpp:17-40 (ContractError, StoreError, FormatError)
 * plus device failures. */
typedef enum {
  FRAG_OK = 0,
  FRAG_E_CONTRACT = 1, /* precondition violation            -> frag::ContractError */
  FRAG_E_STORE = 2,    /* duplicate / missing / capacity     -> frag::StoreError    */
  FRAG_E_FORMAT = 3,   /* bad magic / version / truncation   -> frag::FormatError   */
  FRAG_E_CUDA = 4,     /* CUDA runtime failure or no device                          */
  FRAG_E_OOM = 5       /* device allocation failed                                   */
} frag_status;

/* ModelConfig extended with GQA and Llama-style FFN width. */
typedef struct {
  int32_t layers;     /* D */
  int32_t d_model;    /* hd */
  int32_t n_heads;    /* query heads */
  int32_t n_kv_heads; /* KV heads (== n_heads is the spec's MHA) */
  int32_t head_dim;   /* even */
  int32_t ffn_dim;    /* gated FFN inner width */
  int32_t vocab;
  double rope_base;   /* RotationFrequencies.base */
  float norm_eps;     /* RMSNorm epsilon (1e-5) */
} frag_model_cfg;

typedef struct { uint8_t bytes[16]; } frag_chunk_id; /* Hash128 / ChunkId (common.hpp:103-117) */

typedef struct frag_engine frag_engine;
typedef struct frag_store frag_store;
typedef struct frag_result frag_result;

enum { FRAG_VARIANT_ISOLATED = 0, FRAG_VARIANT_FUSED = 1 }; /* ChunkKVRecord.variant */
/* FRAG_TIER_PEER: the record's pages live in another GPU's store (chunk-
 * partitioned store) and are read over NVLink 5 / NVSwitch. */
enum { FRAG_TIER_GPU = 0, FRAG_TIER_CPU = 1, FRAG_TIER_DISK = 2, FRAG_TIER_PEER = 3 };

/* Read-only view of a ChunkKVRecord. */
typedef struct {
  frag_chunk_id id;
  int32_t n_tok;
  int32_t native_start; /* 1-based position of the record's first token */
  int32_t variant;
  int32_t tier;         /* FRAG_TIER_GPU (this store's HBM) or FRAG_TIER_PEER (another GPU's HBM) */
  uint64_t heat;        /* access count */
  uint64_t last_access; /* store tick of the last fetch */
  uint64_t size_bytes;
  const void* k_dev;    /* [L][n_tok][Hkv][dh] bf16 */
  const void* v_dev;
  const int32_t* tokens_dev; /* [n_tok] token ids (needed by the recompute gather) */
} frag_record_view;

typedef struct {
  int32_t raw_scores;          /* column-sum raw logits instead of joint softmax */
  int32_t all_logits;          /* logits for all question rows (default: last row = first token) */
  int32_t timing;              /* record per-stage device timings (cudaEvents on the stream) */
  const int32_t* inject_crit;  /* optional host list of critical 1-based positions; bypasses the
                                  query-guided selector ("selection-injection" parity mode) */
  int32_t n_inject;
  int32_t logits_on_device;    /* do not copy logits to host (device-resident benchmark leg) */
  int32_t selector;            /* FRAG_SELECT_QUERY_GUIDED (default) or FRAG_SELECT_CACHEBLEND */
  int32_t deviation_layer;     /* CacheBlend: 1-based layer of the deviation (0 -> 2: Delta_KV[:, 2], Eq. 8) */
  int32_t deviation_component; /* CacheBlend: FRAG_DEV_K (default, Delta_KV[:, 2, 1]), FRAG_DEV_V, FRAG_DEV_KV */
  /* Unmatched-chunk fallback (flag-gated): when non-null,
   * fallback_tokens[i] / fallback_lens[i] are the token ids of chunk i (null /
   * 0 for none). A chunk whose record the store does not hold is then
   * prefilled on the fly in isolation (Eq. 5, native_start = n_sys + 1, the
   * tokens must hash to chunk_ids[i]) and inserted into the store before the
   * stitch; without it a missing record is FRAG_E_STORE. */
  const int32_t* const* fallback_tokens;
  const int32_t* fallback_lens;
} frag_reprocess_opts;
/* Critical-token selectors of the reprocessing module: select_query_guided
 * (FusionRAG §3.2) and select_cacheblend (SPEC.md:417-425,
 * Eq. 8: argTopk of the layer-2 K deviation between Full Attention and Full
 * Reuse over cat(S, chunks), lower index on ties). */
enum { FRAG_SELECT_QUERY_GUIDED = 0, FRAG_SELECT_CACHEBLEND = 1 };
enum { FRAG_DEV_K = 0, FRAG_DEV_V = 1, FRAG_DEV_KV = 2 };

typedef struct {
  float stitch_ms;   /* K1 */
  float question_ms; /* question pass through the final-layer Q projection */
  float select_ms;   /* K9 + K10 */
  float sparse_ms;   /* selective-recompute prefill, all layers */
  float lm_head_ms;  /* final norm + K11 + logits copy */
  float total_ms;
  float host_prep_ms; /* host work before the first device launch (always measured) */
} frag_timing;

/* ------------------------------------------------------------------ misc */
FRAG_API const char* frag_last_error(void);
FRAG_API const char* frag_version(void);
/* Presets: "tiny", "llama3-8b", "mistral-7b", "llama3-70b". */
FRAG_API frag_status frag_model_preset(const char* name, frag_model_cfg* out);
/* hash_tokens (common.hpp:122): 128-bit content hash of a token list. */
FRAG_API void frag_hash_tokens(const int32_t* tokens, int32_t n, uint64_t salt, frag_chunk_id* out);
/* Number of device kernels this process has launched through the library. */
FRAG_API uint64_t frag_launch_count(void);
/* Synchronous copy between any two host/device pointers (cudaMemcpyDefault);
 * lets FFI callers read result and record buffers into their own memory. */
FRAG_API frag_status frag_memcpy(void* dst, const void* src, size_t bytes);

/* ------------------------------------------------------------------ engine
 * init_model: weights ~ N(0, 0.02^2) drawn from the splitmix64
 * Rng (common.hpp:45-100), one stream per tensor, rounded to bf16; norm gains 1. */
FRAG_API frag_status frag_engine_create(const frag_model_cfg* cfg, int device, uint64_t seed, frag_engine** out);
FRAG_API frag_status frag_engine_destroy(frag_engine* eng);
FRAG_API frag_status frag_engine_config(const frag_engine* eng, frag_model_cfg* out);
/* Copy one weight tensor in canonical [out][in] layout to a host bf16 buffer.
 * which: 0 emb[V][d] 1 lm_head[V][d] 2 wq 3 wk 4 wv 5 wo 6 w_gate 7 w_up 8 w_down
 *        9 attn_norm 10 ffn_norm 11 final_norm. */
FRAG_API frag_status frag_engine_weight(const frag_engine* eng, int32_t layer, int32_t which, uint16_t* host_out,
                                        size_t n_elems);
FRAG_API uint64_t frag_engine_weight_seed(uint64_t seed, int32_t tensor_id);

/* ------------------------------------------------------------------ store
 * HBM-resident chunk-KV store: put_record, fetch. */
FRAG_API frag_status frag_store_create(const frag_model_cfg* cfg, int device, size_t hbm_bytes, frag_store** out);
FRAG_API frag_status frag_store_destroy(frag_store* st);
/* k/v may be host or device pointers ([L][n_tok][Hkv][dh] bf16); duplicate
 * without overwrite -> FRAG_E_STORE (single-copy invariant). */
FRAG_API frag_status frag_store_put(frag_store* st, const frag_chunk_id* id, const int32_t* tokens, int32_t n_tok,
                                    int32_t native_start, int32_t variant, const void* k_bf16, const void* v_bf16,
                                    int32_t overwrite);
/* heat++, pin; missing id -> FRAG_E_STORE. */
FRAG_API frag_status frag_store_fetch(frag_store* st, const frag_chunk_id* id, frag_record_view* out);
FRAG_API frag_status frag_store_release(frag_store* st, const frag_chunk_id* id);
FRAG_API frag_status frag_store_peek(const frag_store* st, const frag_chunk_id* id, frag_record_view* out);
/* FKVC record files (serialize_record / deserialize_record): magic
 * "FKVC", version u32 = 1, chunk_id[16], variant u8, native_start u32, layers
 * u16, heads u16 (KV heads), head_dim u16, tokens u32, then for every layer K
 * then V, [tokens][heads][head_dim] little-endian fp32. Token ids are not in
 * the file; the loader takes them from the caller. Errors: FRAG_E_FORMAT with
 * frag_last_format_kind() = FRAG_FORMAT_BAD_MAGIC / BAD_VERSION / TRUNCATED /
 * MALFORMED / IO (FormatError::Kind, common.hpp:33). */
typedef struct {
  frag_chunk_id id;
  int32_t variant, native_start, layers, heads, head_dim, tokens;
} frag_fkvc_header;
enum { FRAG_FORMAT_BAD_MAGIC = 0, FRAG_FORMAT_BAD_VERSION = 1, FRAG_FORMAT_TRUNCATED = 2, FRAG_FORMAT_MALFORMED = 3,
       FRAG_FORMAT_IO = 4 };
FRAG_API int32_t frag_last_format_kind(void);
/* Host-only codec: k, v host fp32 [layers][tokens][heads][head_dim]. */
FRAG_API frag_status frag_fkvc_write(const char* path, const frag_fkvc_header* h, const float* k, const float* v);
/* Reads the header (and, if k/v are non-null, the tensors: cap_floats = capacity
 * of each of k and v in floats). */
FRAG_API frag_status frag_fkvc_read(const char* path, frag_fkvc_header* h, float* k, float* v, size_t cap_floats);
/* Write a store record to an FKVC file (bf16 -> fp32, exact). */
FRAG_API frag_status frag_store_save(frag_store* st, const frag_chunk_id* id, const char* path);
/* KVCache loader (DISK -> GPU tier): reads an FKVC file layer
 * by layer into pinned ping-pong buffers while the previous layer is copied
 * H2D and converted to bf16 on `stream`; inserts the record (id from the file)
 * when the copy completes. Safe to call from a loader thread while other
 * threads run frag_reprocess on other streams. */
FRAG_API frag_status frag_store_load(frag_store* st, const char* path, const int32_t* tokens, int32_t n_tok,
                                     int32_t overwrite, void* stream, frag_chunk_id* id_out);
/* Manifest ("JSON file mapping chunk_id -> relative path + variant
 * + native_start"; each entry also lists the chunk's token ids, which FKVC
 * omits): save every record this store owns as <dir>/<chunk id hex>.fkvc plus
 * <dir>/<name> (default "manifest.json"); load every entry of a manifest
 * through frag_store_load (all entries are validated against their files'
 * headers first: FRAG_E_FORMAT Io / Malformed / FKVC kinds, nothing inserted). */
FRAG_API frag_status frag_store_save_manifest(frag_store* st, const char* dir, const char* name, int32_t* n_saved);
FRAG_API frag_status frag_store_load_manifest(frag_store* st, const char* manifest_path, int32_t overwrite,
                                              void* stream, int32_t* n_loaded);
/* Host-only manifest check (no device): parses the manifest and every file
 * header it references; *n_records = number of entries. */
FRAG_API frag_status frag_manifest_validate(const char* manifest_path, int32_t* n_records);
/* Chunk-partitioned store across the GPUs of one box (the
 * spec's single-copy invariant, held across GPUs): each chunk's
 * record lives in exactly one GPU's store (owner = frag_chunk_owner) and the
 * other GPUs read its pages in place over NVLink — K1 (rope_shift_assemble)
 * streams them straight into the local fused cache, so fetch and
 * re-positioning are one pass and no collective runs on the data path.
 *
 * Same process, several devices: after frag_store_attach_peer(local, remote),
 * a fetch that misses `local` is served from `remote` (heat/pins are kept by
 * the owning store; peer access is enabled between the two devices). Records
 * of `remote` are not re-exported through `local` (no transitive lookup).
 * `remote` must outlive `local`.
 *
 * One process per GPU: the owner exports a record (its CUDA IPC memory handle
 * plus metadata in a plain 128-byte struct that any transport can carry, e.g.
 * torch.distributed all_gather_object); every other process imports it as a
 * FRAG_TIER_PEER view. An exported record cannot be overwritten (FRAG_E_STORE);
 * the owning store must outlive its importers (barrier before destroy).
 * Importing a record exported by the same process is a contract error (use
 * attach_peer); importing an id the store already holds needs overwrite. */
typedef struct {
  frag_chunk_id id;
  int32_t n_tok, native_start, variant, owner_device;
  int32_t layers, n_kv_heads, head_dim;
  int32_t owner_pci;         /* owner GPU: PCI domain << 16 | bus << 8 | device (process-independent) */
  uint64_t kv_bytes;         /* K|V allocation size, 2*L*n_tok*Hkv*dh*2 */
  uint64_t owner_pid;        /* exporting process */
  uint8_t ipc_handle[64];    /* cudaIpcMemHandle_t of the K|V allocation */
} frag_peer_record;
/* owner rank of a chunk in a world of n_owners GPUs: little-endian u64 of the
 * first 8 id bytes mod n_owners (ids are content hashes, so this is uniform). */
FRAG_API int32_t frag_chunk_owner(const frag_chunk_id* id, int32_t n_owners);
FRAG_API frag_status frag_store_attach_peer(frag_store* local, frag_store* remote);
FRAG_API frag_status frag_store_export(frag_store* st, const frag_chunk_id* id, frag_peer_record* out);
FRAG_API frag_status frag_store_import(frag_store* st, const frag_peer_record* rec, const int32_t* tokens,
                                       int32_t n_tok, int32_t overwrite);
/* alternative_path_match (§4.1 "progressive
 * backtracking"): a per-store prefix index maps PrefixKey = rolling 128-bit
 * hash over (system-prompt id, ordered chunk ids) to the
 * last chunk of that path. frag_store_register_prefix records that `path`
 * (n >= 1 chunk ids, the record of path[n-1] computed under the preceding
 * ones) is cached; frag_preprocess_isolated registers (sys, [chunk]) itself.
 * frag_store_match walks the context: chunk i matches via PREFIX when the key
 * of (sys, context[0..i]) is registered, else the earliest remaining preceding
 * chunk is dropped until a key hits (ALT_PATH); a chunk whose record exists
 * but no path hits still matches ALT_PATH on its own (alternative-path
 * completeness). Unmatched chunks are simply absent from the
 * output (no error). sys_id: frag_hash_tokens of the system prompt (or null
 * for none). out must hold n entries; *n_out = matches written, in context
 * order. */
enum { FRAG_MATCH_PREFIX = 0, FRAG_MATCH_ALT_PATH = 1 };
typedef struct {
  frag_chunk_id id;
  int32_t matched_via; /* FRAG_MATCH_PREFIX or FRAG_MATCH_ALT_PATH */
  int32_t position;    /* index of the chunk in the context */
  int32_t path_start;  /* first context index of the path that hit (== position for the chunk alone) */
} frag_match;
FRAG_API frag_status frag_store_register_prefix(frag_store* st, const frag_chunk_id* sys_id, const frag_chunk_id* path,
                                                int32_t n);
FRAG_API frag_status frag_store_match(frag_store* st, const frag_chunk_id* sys_id, const frag_chunk_id* context,
                                      int32_t n, frag_match* out, int32_t* n_out);
FRAG_API int64_t frag_store_count(const frag_store* st);
FRAG_API uint64_t frag_store_bytes_used(const frag_store* st);

/* preprocess_isolated (Eq. 5) for one chunk on
 * the GPU: prefill cat(S, C) at positions 1..|S|+|C| and put the record
 * KV[|S|+1:] with native_start = |S|+1. Writes the chunk id (hash_tokens). */
FRAG_API frag_status frag_preprocess_isolated(frag_engine* eng, frag_store* st, const int32_t* sys, int32_t n_sys,
                                              const int32_t* tokens, int32_t n_tok, int32_t overwrite,
                                              frag_chunk_id* id_out);

/* ------------------------------------------------------------------ reprocess
 * A result owns the fused KV cache of one request (the per-request
 * exclusive pages of SPEC.md:148 are the rows recomputed in it) and its
 * logits; it can be reused across requests of at most max_tokens tokens. */
/* preprocess_fused (Eq. 10): prefill C at
 * positions |X|+1.. against cat(KV_S, the listed neighbours' ISOLATED records
 * from `src` stitched consecutively after S), neighbours in the given order
 * (descending similarity), truncated from the tail once their total exceeds
 * `budget` tokens (0 = 2048). Puts a FUSED record (native_start |X|+1) into
 * `dst` (may be `src`; overwrite replaces the ISOLATED record). Missing
 * neighbour -> FRAG_E_STORE naming it. No neighbours -> the ISOLATED K/V. */
FRAG_API frag_status frag_preprocess_fused(frag_engine* eng, frag_store* src, frag_store* dst, const int32_t* sys,
                                          int32_t n_sys, const int32_t* tokens, int32_t n_tok,
                                          const frag_chunk_id* neighbors, int32_t n_neighbors, int32_t budget,
                                          int32_t overwrite, frag_chunk_id* id_out);
FRAG_API frag_status frag_result_create(frag_engine* eng, int32_t max_tokens, frag_result** out);
FRAG_API frag_status frag_result_free(frag_result* res);

/* stitch_full_reuse + select_query_guided + sparse_prefill_and_decode up to the
 * first-token logits. recompute_ratio r: k = floor(r*N + 0.5)
 * critical tokens. stream: cudaStream_t (NULL = legacy default). */
FRAG_API frag_status frag_reprocess(frag_engine* eng, frag_store* st, const int32_t* sys, int32_t n_sys,
                                    const int32_t* question, int32_t n_q, const frag_chunk_id* chunk_ids,
                                    int32_t n_chunks, float recompute_ratio, const frag_reprocess_opts* opts,
                                    void* stream, frag_result* res);
/* Same pipeline with the question tokens already on the device (benchmark leg). */
FRAG_API frag_status frag_reprocess_dev(frag_engine* eng, frag_store* st, const int32_t* sys, int32_t n_sys,
                                        const int32_t* question_dev, int32_t n_q, const frag_chunk_id* chunk_ids,
                                        int32_t n_chunks, float recompute_ratio, const frag_reprocess_opts* opts,
                                        void* stream, frag_result* res);
/* Full Attention prefill (Eq. 2) of cat(S, tokens) with the same kernels: the
 * "full prefill" baseline of BASELINE.json and the r=1 endpoint oracle. */
FRAG_API frag_status frag_full_prefill(frag_engine* eng, const int32_t* sys, int32_t n_sys, const int32_t* tokens,
                                       int32_t n_tok, const frag_reprocess_opts* opts, void* stream,
                                       frag_result* res);

/* Multi-request batching (the scheduler's continuous
 * batching): n_req independent requests reprocessed together.
 * Request b owns rows [b*slot_tokens, b*slot_tokens + T_b) of the result's
 * fused cache (result capacity >= n_req * slot_tokens, T_b <= slot_tokens);
 * the question pass and the sparse pass run once over all requests' rows, so
 * every weight matrix streams once per batch, while attention, scoring and
 * top-k stay per request. Each request's fused KV rows, critical set and
 * first-token logits equal those of frag_reprocess on the same inputs.
 * Logits: n_req rows (row b = request b's last question token). Options:
 * timing / raw_scores / logits_on_device; no injection, no CacheBlend, no
 * all_logits; frag_decode is not available after a batch. */
typedef struct {
  const int32_t* sys;
  int32_t n_sys;
  const int32_t* question;
  int32_t n_q;
  const frag_chunk_id* chunk_ids;
  int32_t n_chunks;
  float recompute_ratio;
} frag_request;
FRAG_API frag_status frag_reprocess_batch(frag_engine* eng, frag_store* st, const frag_request* reqs, int32_t n_req,
                                          int32_t slot_tokens, const frag_reprocess_opts* opts, void* stream,
                                          frag_result* res);
/* Critical positions (1-based, ascending) of request b of the last batch;
 * returns their count (or -1), writing up to cap of them when host_out != NULL. */
FRAG_API int32_t frag_result_batch_crit(const frag_result* res, int32_t b, int32_t* host_out, int32_t cap);

/* kv_deviation (Eq. 7): Full Reuse (the
 * stitched records) against Full Attention over cat(S, chunks) through the
 * first n_layers layers; dev_host receives [N][n_layers][2] fp32 (K, V sums of
 * squared per-dim differences, N = total chunk tokens). Afterwards `res` holds
 * the Full-Reuse stitched cache of the context (question rows unset). */
FRAG_API frag_status frag_kv_deviation(frag_engine* eng, frag_store* st, const int32_t* sys, int32_t n_sys,
                                       const frag_chunk_id* chunk_ids, int32_t n_chunks, int32_t n_layers,
                                       void* stream, frag_result* res, float* dev_host);

/* sparse_prefill_and_decode, decode half: greedy decoding
 * continuing the last frag_reprocess / frag_full_prefill of `res`. Token 0 is
 * the argmax of the last logits row (lowest index on ties); each further token
 * is one single-row step at the next position whose K/V are appended to the
 * result's fused cache (the request's exclusive pages; records untouched).
 * Needs result capacity >= T + max_new_tokens - 1. Writes max_new_tokens ids
 * to host tokens_out; afterwards the result holds the last step's logits. */
FRAG_API frag_status frag_decode(frag_engine* eng, frag_result* res, int32_t max_new_tokens, void* stream,
                                 int32_t* tokens_out);
FRAG_API frag_status frag_result_sync(frag_result* res);
/* Fused cache: device pointers [L][max_tokens][Hkv][dh] bf16 (rows [0, T) valid,
 * T = tokens in the prompt, plus decoded tokens). With shared V pages (the
 * default for query-guided requests) V is read in place from the records and
 * the request's exclusive slots; asking for v_dev assembles that view into the
 * result's V buffer (synchronous, after the request's stream work). */
FRAG_API frag_status frag_result_fused_kv(const frag_result* res, const void** k_dev, const void** v_dev,
                                          int32_t* n_tokens);
/* Logits fp32 [rows][V]; host pointer (or device pointer with logits_on_device). */
FRAG_API frag_status frag_result_logits(const frag_result* res, const float** logits, int32_t* rows,
                                        int32_t* vocab, int32_t on_device);
/* Critical positions (1-based, ascending) chosen for the last request. */
FRAG_API int32_t frag_result_crit(const frag_result* res, int32_t* host_out, int32_t cap);
/* Stage times of the last call (0 unless it set opts.timing; timed calls run
 * eagerly, untimed ones replay a CUDA graph) and its host prep time. */
FRAG_API frag_status frag_result_timing(const frag_result* res, frag_timing* out);
/* Debug views for parity tests: final-layer question queries fp32 [n_q][Hq][dh]
 * and the per-token query-guided scores fp32 [N] (device pointers). */
FRAG_API frag_status frag_result_debug(const frag_result* res, const float** q_final_dev, const float** scores_dev,
                                       int32_t* n_q, int32_t* n_chunk_tokens);

/* ------------------------------------------------------------------ profiling
 * Per-kernel-class device timing (cudaEvents around each launch on the
 * launching stream) for the bench roofline. class: 0 tensor-bound GEMM
 * (K4/K7/K8/K11 at > 128 rows), 1 attention (K6), 2 stitch (K1), 3 norms/gather
 * (K2/K3), 4 select (K9/K10), 5 weight-streaming GEMM (<= 128 rows: the
 * question pass and lm_head rows; algorithmic bytes = weight bytes), 6 the
 * gate/up projection GEMM alone at > 128 rows (a subset of class 0: the
 * single largest kernel, the bench's roofline kernel), 7 the shared-V window
 * fills of the large passes (records' V of one layer copied into the staging
 * window; algorithmic bytes = read + write). */
FRAG_API frag_status frag_engine_profile(frag_engine* eng, int32_t enable);
/* Sums over launches since the last reset (call after frag_result_sync):
 * device ms, algorithmic FLOPs, algorithmic bytes, launch count. */
FRAG_API frag_status frag_engine_profile_read(frag_engine* eng, int32_t klass, double* ms, double* flops,
                                              double* bytes, int64_t* launches, int32_t reset);
/* Limit of the persistent kernels' inter-CTA waits (a grid that is not
 * co-resident -- another context holding SMs -- abandons the wait after this
 * long and the call returns FRAG_E_CUDA instead of hanging). Process wide;
 * default FRAG_SPIN_LIMIT_MS or 2000 ms; ms <= 0 restores the default.
 * Returns the previous limit in ms. */
FRAG_API double frag_set_spin_limit_ms(double ms);
/* Shared V pages: on (default, FRAG_SHARED_V=0 turns it
 * off) query-guided requests read their chunks' V rows in place from the
 * records and keep only their fresh rows in exclusive slots; off: every request
 * copies V into a private fused cache (the layout of frag_full_prefill).
 * on = 1 / 0 sets, -1 only queries; returns the previous setting. Process wide. */
FRAG_API int32_t frag_set_shared_v(int32_t on);
/* Device memory held by a result (fused K, V view or exclusive V slots, plans
 * and workspaces) and whether its last request used shared V pages. */
FRAG_API frag_status frag_result_memory(const frag_result* res, uint64_t* device_bytes, int32_t* shared_v);

/* ------------------------------------------------------------------ kernels
 * Kernel-level entry points over device pointers (parity tests, bench roofline). */
/* C[M,N] = A[M,K] B[N,K]^T, bf16 in, epi 0: bf16 out, 1: fp32 out, 2: fp32 C += . */
FRAG_API frag_status frag_kernel_gemm(const void* a, const void* b, void* c, int32_t M, int32_t N, int32_t K,
                                      int32_t epi, int32_t force_bn, void* stream);
/* K1 on one record: dst[L][n][Hkv][dh] = shift_rope(src, native_start -> target_start). */
FRAG_API frag_status frag_kernel_rope_shift(const void* k_src, void* k_dst, int32_t L, int32_t n_tok, int32_t Hkv,
                                            int32_t dh, int32_t native_start, int32_t target_start,
                                            double rope_base, void* stream);
/* K9+K10 on given final-layer queries q[nq][Hq][dh] fp32 and keys k[N][Hkv][dh] bf16. */
FRAG_API frag_status frag_kernel_qg_select(const float* q, const void* k, int32_t nq, int32_t Hq, int32_t Hkv,
                                           int32_t dh, int32_t n_keys, int32_t k_sel, int32_t raw,
                                           float* scores_dev, int32_t* sel_dev, void* stream);
/* K6: q[M][Hq][dh], k/v [T][Hkv][dh] bf16, rows[M] ascending query rows -> out[M][Hq][dh]. */
FRAG_API frag_status frag_kernel_attention(const void* q, const void* k, const void* v, const int32_t* rows,
                                           void* out, int32_t M, int32_t T, int32_t Hq, int32_t Hkv, int32_t dh,
                                           int32_t split_keys, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FRAG_C_H */
