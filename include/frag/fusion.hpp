// frag::fusion — C++ API of the B200 reprocessing path (RAII over frag_c.h).
//
// Mirrors the reference's operation surface for the online stage:
//   ChunkStore::put_record / fetch
//   Engine::preprocess_isolated             SPEC.md:344-352 (Eq. 5)
//   Engine::preprocess_fused                SPEC.md:353-361 (Eq. 10)
//   Engine::reprocess                        stitch_full_reuse + select_query_guided +
//                                            sparse_prefill_and_decode to the first token
//
//   Engine::full_prefill                     Eq. 2 Full Attention with the same kernels
//   Engine::decode                           greedy decoding over the fused cache
// Status codes from the C ABI are re-thrown as the reference's exception
// classes (common.hpp:17-40): ContractError, StoreError, FormatError.
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "frag/core.hpp"
#include "frag/frag_c.h"

namespace frag {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(frag_status s) {
  if (s == FRAG_OK) return;
  const std::string m = frag_last_error();
  switch (s) {
    case FRAG_E_CONTRACT: throw ContractError(m);
    case FRAG_E_STORE: throw StoreError(m);
    case FRAG_E_FORMAT: {
      // the library's thread-local kind of the last FRAG_E_FORMAT (frag_c.h) ->
      // the reference's FormatError::Kind (common.hpp:33)
      FormatError::Kind k = FormatError::Kind::Malformed;
      switch (frag_last_format_kind()) {
        case FRAG_FORMAT_BAD_MAGIC: k = FormatError::Kind::BadMagic; break;
        case FRAG_FORMAT_BAD_VERSION: k = FormatError::Kind::BadVersion; break;
        case FRAG_FORMAT_TRUNCATED: k = FormatError::Kind::Truncated; break;
        case FRAG_FORMAT_IO: k = FormatError::Kind::Io; break;
        default: break;
      }
      throw FormatError(k, m);
    }
    case FRAG_E_OOM: throw std::bad_alloc();
    default: throw CudaError(m);
  }
}

inline frag_chunk_id to_c(const ChunkId& id) {
  frag_chunk_id c;
  std::memcpy(c.bytes, id.bytes.data(), 16);
  return c;
}
inline ChunkId from_c(const frag_chunk_id& c) {
  ChunkId id;
  std::memcpy(id.bytes.data(), c.bytes, 16);
  return id;
}

inline frag_model_cfg preset(const std::string& name) {
  frag_model_cfg c{};
  check(frag_model_preset(name.c_str(), &c));
  return c;
}

class ChunkStore {
 public:
  ChunkStore(const frag_model_cfg& cfg, int device = 0, size_t hbm_bytes = 0) {
    check(frag_store_create(&cfg, device, hbm_bytes, &h_));
  }
  ~ChunkStore() { frag_store_destroy(h_); }
  ChunkStore(const ChunkStore&) = delete;
  ChunkStore& operator=(const ChunkStore&) = delete;

  // put_record: k/v host or device [L][n][Hkv][dh] bf16 bits.
  void put_record(const ChunkId& id, std::span<const Token> tokens, Pos native_start, const void* k_bf16,
                  const void* v_bf16, int variant = FRAG_VARIANT_ISOLATED, bool overwrite = false) {
    const frag_chunk_id c = to_c(id);
    check(frag_store_put(h_, &c, tokens.data(), static_cast<int32_t>(tokens.size()), native_start, variant, k_bf16,
                         v_bf16, overwrite ? 1 : 0));
  }
  // fetch: heat++, pinned until release().
  frag_record_view fetch(const ChunkId& id) {
    const frag_chunk_id c = to_c(id);
    frag_record_view v{};
    check(frag_store_fetch(h_, &c, &v));
    return v;
  }
  void release(const ChunkId& id) {
    const frag_chunk_id c = to_c(id);
    check(frag_store_release(h_, &c));
  }
  size_t size() const { return static_cast<size_t>(frag_store_count(h_)); }
  uint64_t bytes_used() const { return frag_store_bytes_used(h_); }
  frag_store* handle() const { return h_; }

  // Chunk-partitioned store: owner rank of a chunk, a
  // same-process peer store on another GPU (misses served in place over
  // NVLink), and the cross-process CUDA-IPC export / import of one record.
  static int owner_of(const ChunkId& id, int n_owners) {
    const frag_chunk_id c = to_c(id);
    return frag_chunk_owner(&c, n_owners);
  }
  void attach_peer(ChunkStore& remote) { check(frag_store_attach_peer(h_, remote.h_)); }
  // alternative_path_match: matches in context order; unmatched chunks absent
  void register_prefix(std::span<const ChunkId> path, const ChunkId* sys_id = nullptr) {
    std::vector<frag_chunk_id> p;
    for (const auto& c : path) p.push_back(to_c(c));
    const frag_chunk_id s = sys_id ? to_c(*sys_id) : frag_chunk_id{};
    check(frag_store_register_prefix(h_, sys_id ? &s : nullptr, p.data(), static_cast<int32_t>(p.size())));
  }
  std::vector<frag_match> match(std::span<const ChunkId> context, const ChunkId* sys_id = nullptr) {
    std::vector<frag_chunk_id> c;
    for (const auto& x : context) c.push_back(to_c(x));
    std::vector<frag_match> out(c.size());
    int32_t n = 0;
    const frag_chunk_id s = sys_id ? to_c(*sys_id) : frag_chunk_id{};
    check(frag_store_match(h_, sys_id ? &s : nullptr, c.data(), static_cast<int32_t>(c.size()), out.data(), &n));
    out.resize(n);
    return out;
  }
  frag_peer_record export_record(const ChunkId& id) {
    const frag_chunk_id c = to_c(id);
    frag_peer_record pr{};
    check(frag_store_export(h_, &c, &pr));
    return pr;
  }
  void import_record(const frag_peer_record& pr, std::span<const Token> tokens, bool overwrite = false) {
    check(frag_store_import(h_, &pr, tokens.data(), static_cast<int32_t>(tokens.size()), overwrite ? 1 : 0));
  }

 private:
  frag_store* h_ = nullptr;
};

class Engine;

// Shared V pages on / off for the process (frag_set_shared_v); returns the previous setting.
inline bool set_shared_v(bool on) { return frag_set_shared_v(on ? 1 : 0) != 0; }

// Fused KV cache + first-token logits of one request; reusable.
class Result {
 public:
  Result(Engine& e, int max_tokens);
  ~Result() { frag_result_free(h_); }
  Result(const Result&) = delete;
  Result& operator=(const Result&) = delete;

  std::vector<float> logits() const {
    const float* p = nullptr;
    int32_t rows = 0, vocab = 0;
    check(frag_result_logits(h_, &p, &rows, &vocab, 0));
    return std::vector<float>(p, p + static_cast<size_t>(rows) * vocab);
  }
  Token first_token() const {  // greedy argmax of the last question row
    const float* p = nullptr;
    int32_t rows = 0, vocab = 0;
    check(frag_result_logits(h_, &p, &rows, &vocab, 0));
    const float* last = p + static_cast<size_t>(rows - 1) * vocab;
    int32_t best = 0;
    for (int32_t i = 1; i < vocab; ++i)
      if (last[i] > last[best]) best = i;
    return best;
  }
  std::vector<Pos> critical_positions() const {
    const int32_t k = frag_result_crit(h_, nullptr, 0);
    std::vector<Pos> out(k > 0 ? k : 0);
    if (k > 0) frag_result_crit(h_, out.data(), k);
    return out;
  }
  std::vector<Pos> batch_critical_positions(int b) const {
    const int32_t k = frag_result_batch_crit(h_, b, nullptr, 0);
    if (k < 0) throw ContractError("no such request in the last batch");
    std::vector<Pos> out(k);
    if (k > 0) frag_result_batch_crit(h_, b, out.data(), k);
    return out;
  }
  frag_timing timing() const {
    frag_timing t{};
    check(frag_result_timing(h_, &t));
    return t;
  }
  // device pointers [L][max_tokens][Hkv][dh] bf16, rows [0, tokens) valid; with
  // shared V pages the V view is assembled from the records on this call
  void fused_kv(const void** k, const void** v, int32_t* tokens) const { check(frag_result_fused_kv(h_, k, v, tokens)); }
  // device bytes held by the result and whether its last request read V in place
  std::pair<uint64_t, bool> memory() const {
    uint64_t b = 0;
    int32_t sv = 0;
    check(frag_result_memory(h_, &b, &sv));
    return {b, sv != 0};
  }
  frag_result* handle() const { return h_; }

 private:
  frag_result* h_ = nullptr;
};

class Engine {
 public:
  // init_model: seeded random weights, bf16 on `device`.
  Engine(const frag_model_cfg& cfg, int device = 0, uint64_t seed = 1234) {
    check(frag_engine_create(&cfg, device, seed, &h_));
  }
  ~Engine() { frag_engine_destroy(h_); }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  frag_model_cfg config() const {
    frag_model_cfg c{};
    check(frag_engine_config(h_, &c));
    return c;
  }

  ChunkId preprocess_isolated(ChunkStore& st, std::span<const Token> chunk, std::span<const Token> system = {},
                              bool overwrite = false) {
    frag_chunk_id id{};
    check(frag_preprocess_isolated(h_, st.handle(), system.data(), static_cast<int32_t>(system.size()), chunk.data(),
                                   static_cast<int32_t>(chunk.size()), overwrite ? 1 : 0, &id));
    return from_c(id);
  }

  // preprocess_fused (Eq. 10): FUSED record of `chunk` prefilled
  // against KV_S + the neighbours' ISOLATED records (descending similarity).
  ChunkId preprocess_fused(ChunkStore& src, std::span<const Token> chunk, std::span<const ChunkId> neighbors,
                           std::span<const Token> system = {}, ChunkStore* dst = nullptr, int budget = 2048,
                           bool overwrite = false) {
    std::vector<frag_chunk_id> nb;
    nb.reserve(neighbors.size());
    for (const auto& n : neighbors) nb.push_back(to_c(n));
    frag_chunk_id id{};
    check(frag_preprocess_fused(h_, src.handle(), (dst ? dst : &src)->handle(), system.data(),
                                static_cast<int32_t>(system.size()), chunk.data(), static_cast<int32_t>(chunk.size()),
                                nb.data(), static_cast<int32_t>(nb.size()), budget, overwrite ? 1 : 0, &id));
    return from_c(id);
  }

  // reprocess(question, chunk_ids, recompute_ratio) -> fused KV + logits
  void reprocess(ChunkStore& st, std::span<const Token> question, std::span<const ChunkId> chunk_ids, float ratio,
                 Result& out, std::span<const Token> system = {}, const frag_reprocess_opts* opts = nullptr,
                 void* cuda_stream = nullptr) {
    std::vector<frag_chunk_id> ids;
    ids.reserve(chunk_ids.size());
    for (const auto& c : chunk_ids) ids.push_back(to_c(c));
    check(frag_reprocess(h_, st.handle(), system.data(), static_cast<int32_t>(system.size()), question.data(),
                         static_cast<int32_t>(question.size()), ids.data(), static_cast<int32_t>(ids.size()), ratio,
                         opts, cuda_stream, out.handle()));
  }

  // kv_deviation (Eq. 7): [N][n_layers][2] K/V deviation between
  // Full Attention and Full Reuse; select_cacheblend is reprocess() with
  // opts->selector = FRAG_SELECT_CACHEBLEND.
  std::vector<float> kv_deviation(ChunkStore& st, std::span<const ChunkId> chunk_ids, Result& scratch,
                                  std::span<const Token> system = {}, int n_layers = 2, void* cuda_stream = nullptr) {
    std::vector<frag_chunk_id> ids;
    size_t n = 0;
    for (const auto& c : chunk_ids) {
      ids.push_back(to_c(c));
      frag_record_view v{};
      check(frag_store_peek(st.handle(), &ids.back(), &v));
      n += static_cast<size_t>(v.n_tok);
    }
    std::vector<float> dev(n * static_cast<size_t>(n_layers) * 2);
    check(frag_kv_deviation(h_, st.handle(), system.data(), static_cast<int32_t>(system.size()), ids.data(),
                            static_cast<int32_t>(ids.size()), n_layers, cuda_stream, scratch.handle(), dev.data()));
    return dev;
  }

  // Multi-request batching (frag_reprocess_batch): request b uses fused-cache
  // rows [b * slot_tokens, ...) of `out`; logits row b = request b's first token.
  struct Request {
    std::span<const Token> question;
    std::span<const ChunkId> chunk_ids;
    float recompute_ratio = 0.15f;
    std::span<const Token> system = {};
  };
  void reprocess_batch(ChunkStore& st, std::span<const Request> reqs, Result& out, int slot_tokens,
                       const frag_reprocess_opts* opts = nullptr, void* cuda_stream = nullptr) {
    std::vector<std::vector<frag_chunk_id>> ids(reqs.size());
    std::vector<frag_request> cr(reqs.size());
    for (size_t b = 0; b < reqs.size(); ++b) {
      for (const auto& c : reqs[b].chunk_ids) ids[b].push_back(to_c(c));
      cr[b] = frag_request{reqs[b].system.data(), static_cast<int32_t>(reqs[b].system.size()),
                           reqs[b].question.data(), static_cast<int32_t>(reqs[b].question.size()), ids[b].data(),
                           static_cast<int32_t>(ids[b].size()), reqs[b].recompute_ratio};
    }
    check(frag_reprocess_batch(h_, st.handle(), cr.data(), static_cast<int32_t>(cr.size()), slot_tokens, opts,
                               cuda_stream, out.handle()));
  }

  void full_prefill(std::span<const Token> tokens, Result& out, std::span<const Token> system = {},
                    const frag_reprocess_opts* opts = nullptr, void* cuda_stream = nullptr) {
    check(frag_full_prefill(h_, system.data(), static_cast<int32_t>(system.size()), tokens.data(),
                            static_cast<int32_t>(tokens.size()), opts, cuda_stream, out.handle()));
  }

  // Greedy decoding after reprocess / full_prefill (sparse_prefill_and_decode,
  // SPEC.md:435-438): max_new_tokens ids; decoded K/V appended to `res`.
  std::vector<Token> decode(Result& res, int max_new_tokens, void* cuda_stream = nullptr) {
    std::vector<Token> out(max_new_tokens > 0 ? max_new_tokens : 0);
    check(frag_decode(h_, res.handle(), max_new_tokens, cuda_stream, out.data()));
    return out;
  }

  frag_engine* handle() const { return h_; }

 private:
  frag_engine* h_ = nullptr;
};

inline Result::Result(Engine& e, int max_tokens) { check(frag_result_create(e.handle(), max_tokens, &h_)); }

}  // namespace frag
