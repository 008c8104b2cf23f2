// extern "C" boundary (include/frag/frag_c.h). Every entry point converts the
// internal exceptions into frag_status codes + a thread-local message, so no
// C++ exception ever crosses the ABI.
#include <cmath>
#include <cstring>
#include <mutex>
#include <new>
#include <string>

#include "engine.h"

struct frag_engine {
  fragimpl::Engine* e;
};
struct frag_store {
  fragimpl::Store* s;
};
struct frag_result {
  fragimpl::Result* r;
};

namespace fragimpl {

thread_local std::string t_last_error;
thread_local int t_format_kind = -1;

void set_last_error(const std::string& m) { t_last_error = m; }

[[noreturn]] void fail(frag_status code, const std::string& msg) { throw Error{code, msg}; }
[[noreturn]] void fail_format(int kind, const std::string& msg) { throw Error{FRAG_E_FORMAT, msg, kind}; }

namespace {
template <class F>
frag_status guard(F&& f) {
  try {
    f();
    return FRAG_OK;
  } catch (const Error& e) {
    set_last_error(e.msg);
    t_format_kind = e.format_kind;
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return FRAG_E_OOM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return FRAG_E_CONTRACT;
  } catch (...) {
    set_last_error("unknown error");
    return FRAG_E_CONTRACT;
  }
}
void need(bool ok, const char* m) {
  if (!ok) fail(FRAG_E_CONTRACT, m);
}
}  // namespace

}  // namespace fragimpl

using namespace fragimpl;

extern "C" {

FRAG_API const char* frag_last_error(void) { return t_last_error.c_str(); }
FRAG_API int32_t frag_last_format_kind(void) { return t_format_kind; }

FRAG_API frag_status frag_fkvc_write(const char* path, const frag_fkvc_header* h, const float* k, const float* v) {
  return guard([&] {
    need(path && h && k && v, "null argument");
    fkvc_write(path, *h, k, v);
  });
}

FRAG_API frag_status frag_fkvc_read(const char* path, frag_fkvc_header* h, float* k, float* v, size_t cap_floats) {
  return guard([&] {
    need(path && h, "null argument");
    fkvc_read(path, h, k, v, cap_floats);
  });
}
FRAG_API const char* frag_version(void) { return "fusionrag-b200 0.1 (sm_100a)"; }

FRAG_API frag_status frag_model_preset(const char* name, frag_model_cfg* out) {
  return guard([&] {
    need(name && out, "null argument");
    const std::string n(name);
    frag_model_cfg c{};
    c.norm_eps = 1e-5f;
    if (n == "tiny") {  // SPEC.md:81 defaults scaled to BASELINE.json configs[0]
      c = {2, 256, 4, 4, 64, 1024, 256, 1e4, 1e-5f};
    } else if (n == "llama3-8b") {
      c = {32, 4096, 32, 8, 128, 14336, 128256, 5e5, 1e-5f};
    } else if (n == "mistral-7b") {
      c = {32, 4096, 32, 8, 128, 14336, 32768, 1e6, 1e-5f};
    } else if (n == "llama3-70b") {
      c = {80, 8192, 64, 8, 128, 28672, 128256, 5e5, 1e-5f};
    } else {
      fail(FRAG_E_CONTRACT, "unknown preset '" + n + "'");
    }
    *out = c;
  });
}

FRAG_API void frag_hash_tokens(const int32_t* tokens, int32_t n, uint64_t salt, frag_chunk_id* out) {
  if (!out) return;
  hash_tokens(tokens, n < 0 ? 0 : n, salt, out);
}

FRAG_API uint64_t frag_launch_count(void) { return g_launches.load(); }

FRAG_API double frag_set_spin_limit_ms(double ms) {
  const double prev = (double)fragk::spin_limit_ns() / 1e6;
  if (ms <= 0) {
    const char* e = std::getenv("FRAG_SPIN_LIMIT_MS");
    ms = e && std::atof(e) > 0 ? std::atof(e) : 2000.0;
  }
  fragk::set_spin_limit_ns((unsigned long long)(ms * 1e6));
  fragimpl::g_alloc_epoch++;  // captured request graphs hold the old limit in their kernel parameters
  return prev;
}

FRAG_API int32_t frag_set_shared_v(int32_t on) {
  const int32_t prev = fragimpl::set_shared_v(on);
  if (on >= 0 && on != prev) fragimpl::g_alloc_epoch++;  // request graphs captured the other layout
  return prev;
}

FRAG_API frag_status frag_result_memory(const frag_result* res, uint64_t* device_bytes, int32_t* shared_v) {
  return guard([&] {
    need(res, "null result");
    const Result* r = res->r;
    if (device_bytes) *device_bytes = result_device_bytes(r);
    if (shared_v) *shared_v = r->vshared ? 1 : 0;
  });
}

FRAG_API frag_status frag_memcpy(void* dst, const void* src, size_t bytes) {
  return guard([&] {
    need(dst && src, "null argument");
    check_cuda(cudaMemcpy(dst, src, bytes, cudaMemcpyDefault), "frag_memcpy");
  });
}

// ---------------------------------------------------------------- engine
FRAG_API frag_status frag_engine_create(const frag_model_cfg* cfg, int device, uint64_t seed, frag_engine** out) {
  return guard([&] {
    need(cfg && out, "null argument");
    *out = nullptr;
    Engine* e = engine_create(*cfg, device, seed);
    *out = new frag_engine{e};
  });
}

FRAG_API frag_status frag_engine_destroy(frag_engine* eng) {
  return guard([&] {
    if (!eng) return;
    {
      DeviceGuard dg(eng->e->device);
      cudaDeviceSynchronize();
      delete eng->e;
    }
    delete eng;
  });
}

FRAG_API frag_status frag_engine_config(const frag_engine* eng, frag_model_cfg* out) {
  return guard([&] {
    need(eng && out, "null argument");
    *out = eng->e->cfg;
  });
}

FRAG_API uint64_t frag_engine_weight_seed(uint64_t seed, int32_t tensor_id) { return weight_seed(seed, tensor_id); }

FRAG_API frag_status frag_engine_weight(const frag_engine* eng, int32_t layer, int32_t which, uint16_t* host_out,
                                        size_t n_elems) {
  return guard([&] {
    need(eng && host_out, "null argument");
    Engine* e = eng->e;
    const auto& c = e->cfg;
    const size_t d = c.d_model, V = c.vocab, F = c.ffn_dim, qc = (size_t)c.n_heads * c.head_dim,
                 kc = (size_t)c.n_kv_heads * c.head_dim;
    DeviceGuard dg(e->device);
    auto copy_rows = [&](const bf16* base, size_t rows, size_t cols, size_t row0) {
      need(n_elems >= rows * cols, "output buffer too small");
      check_cuda(cudaMemcpy(host_out, base + row0 * cols, rows * cols * sizeof(bf16), cudaMemcpyDeviceToHost),
                 "weight D2H");
    };
    if (which == 0) return copy_rows(e->emb, V, d, 0);
    if (which == 1) return copy_rows(e->lm_head, V, d, 0);
    if (which == 11) return copy_rows(e->final_norm, 1, d, 0);
    need(layer >= 0 && layer < c.layers, "layer out of range");
    const auto& L = e->layers[layer];
    switch (which) {
      case 2: return copy_rows(L.wqkv, qc, d, 0);
      case 3: return copy_rows(L.wqkv, kc, d, qc);
      case 4: return copy_rows(L.wqkv, kc, d, qc + kc);
      case 5: return copy_rows(L.wo, d, qc, 0);
      case 6:
      case 7: {
        // un-interleave the 32-row gate/up blocks
        need(n_elems >= F * d, "output buffer too small");
        std::vector<uint16_t> packed(2 * F * d);
        check_cuda(cudaMemcpy(packed.data(), L.wgu, packed.size() * 2, cudaMemcpyDeviceToHost), "weight D2H");
        const size_t off = which == 6 ? 0 : 32;
        for (size_t r = 0; r < F; ++r)
          std::memcpy(host_out + r * d, packed.data() + ((r / 32) * 64 + off + r % 32) * d, d * 2);
        return;
      }
      case 8: return copy_rows(L.wd, d, F, 0);
      case 9: return copy_rows(L.attn_norm, 1, d, 0);
      case 10: return copy_rows(L.ffn_norm, 1, d, 0);
    }
    fail(FRAG_E_CONTRACT, "unknown weight id");
  });
}

FRAG_API frag_status frag_engine_profile(frag_engine* eng, int32_t enable) {
  return guard([&] {
    need(eng, "null engine");
    eng->e->prof.collect();
    eng->e->prof.on = enable != 0;
  });
}

FRAG_API frag_status frag_engine_profile_read(frag_engine* eng, int32_t klass, double* ms, double* flops,
                                              double* bytes, int64_t* launches, int32_t reset) {
  return guard([&] {
    need(eng, "null engine");
    need(klass >= 0 && klass < KC_N, "profile class out of range");
    Profiler& p = eng->e->prof;
    DeviceGuard dg(eng->e->device);
    p.collect();
    if (ms) *ms = p.ms[klass];
    if (flops) *flops = p.flops[klass];
    if (bytes) *bytes = p.bytes[klass];
    if (launches) *launches = p.launches[klass];
    if (reset) p.reset();
  });
}

// ---------------------------------------------------------------- store
FRAG_API frag_status frag_store_create(const frag_model_cfg* cfg, int device, size_t hbm_bytes, frag_store** out) {
  return guard([&] {
    need(cfg && out, "null argument");
    *out = new frag_store{store_create(*cfg, device, hbm_bytes)};
  });
}

FRAG_API frag_status frag_store_destroy(frag_store* st) {
  return guard([&] {
    if (!st) return;
    {
      DeviceGuard dg(st->s->device);
      cudaDeviceSynchronize();
      delete st->s;
    }
    delete st;
  });
}

FRAG_API frag_status frag_store_put(frag_store* st, const frag_chunk_id* id, const int32_t* tokens, int32_t n_tok,
                                    int32_t native_start, int32_t variant, const void* k_bf16, const void* v_bf16,
                                    int32_t overwrite) {
  return guard([&] {
    need(st && id, "null argument");
    store_put(st->s, *id, tokens, n_tok, native_start, variant, k_bf16, v_bf16, overwrite != 0);
  });
}

static void fill_view(const Record* r, frag_record_view* out) {
  out->id = r->id;
  out->n_tok = r->n_tok;
  out->native_start = r->native_start;
  out->variant = r->variant;
  out->tier = r->tier;
  out->heat = r->heat;
  out->last_access = r->last_access;
  out->size_bytes = r->bytes;
  out->k_dev = r->k();
  out->v_dev = r->v();
  out->tokens_dev = r->tok.as<int32_t>();
}

FRAG_API frag_status frag_store_fetch(frag_store* st, const frag_chunk_id* id, frag_record_view* out) {
  return guard([&] {
    need(st && id && out, "null argument");
    Record* r = store_fetch(st->s, *id);
    std::shared_lock<std::shared_mutex> g(st->s->mu);
    fill_view(r, out);
  });
}

FRAG_API frag_status frag_store_release(frag_store* st, const frag_chunk_id* id) {
  return guard([&] {
    need(st && id, "null argument");
    store_release(st->s, *id);
  });
}

FRAG_API frag_status frag_store_peek(const frag_store* st, const frag_chunk_id* id, frag_record_view* out) {
  return guard([&] {
    need(st && id && out, "null argument");
    std::vector<Store*> stores{st->s};
    {
      std::shared_lock<std::shared_mutex> g(st->s->mu);
      stores.insert(stores.end(), st->s->peers.begin(), st->s->peers.end());
    }
    for (Store* s : stores) {  // local index first, then attached peers (as fetch)
      std::shared_lock<std::shared_mutex> g(s->mu);
      auto it = s->recs.find(key_of(*id));
      if (it != s->recs.end()) {
        fill_view(it->second.get(), out);
        return;
      }
    }
    fail(FRAG_E_STORE, "missing chunk record");
  });
}

FRAG_API frag_status frag_store_save(frag_store* st, const frag_chunk_id* id, const char* path) {
  return guard([&] {
    need(st && id && path, "null argument");
    store_save(st->s, *id, path);
  });
}

FRAG_API frag_status frag_store_load(frag_store* st, const char* path, const int32_t* tokens, int32_t n_tok,
                                     int32_t overwrite, void* stream, frag_chunk_id* id_out) {
  return guard([&] {
    need(st && path && tokens, "null argument");
    store_load(st->s, path, tokens, n_tok, overwrite != 0, static_cast<cudaStream_t>(stream), id_out);
  });
}

FRAG_API frag_status frag_store_save_manifest(frag_store* st, const char* dir, const char* name, int32_t* n_saved) {
  return guard([&] {
    need(st && dir, "null argument");
    const int n = manifest_save(st->s, dir, name);
    if (n_saved) *n_saved = n;
  });
}

FRAG_API frag_status frag_store_load_manifest(frag_store* st, const char* manifest_path, int32_t overwrite,
                                              void* stream, int32_t* n_loaded) {
  return guard([&] {
    need(st && manifest_path, "null argument");
    const int n = manifest_load(st->s, manifest_path, overwrite != 0, static_cast<cudaStream_t>(stream));
    if (n_loaded) *n_loaded = n;
  });
}

FRAG_API frag_status frag_manifest_validate(const char* manifest_path, int32_t* n_records) {
  return guard([&] {
    need(manifest_path, "null argument");
    const auto es = manifest_read(manifest_path);
    if (n_records) *n_records = (int32_t)es.size();
  });
}

FRAG_API int32_t frag_chunk_owner(const frag_chunk_id* id, int32_t n_owners) {
  if (!id || n_owners < 1) return -1;
  return chunk_owner(*id, n_owners);
}

FRAG_API frag_status frag_store_attach_peer(frag_store* local, frag_store* remote) {
  return guard([&] {
    need(local && remote, "null argument");
    store_attach_peer(local->s, remote->s);
  });
}

FRAG_API frag_status frag_store_export(frag_store* st, const frag_chunk_id* id, frag_peer_record* out) {
  return guard([&] {
    need(st && id && out, "null argument");
    store_export(st->s, *id, out);
  });
}

FRAG_API frag_status frag_store_import(frag_store* st, const frag_peer_record* rec, const int32_t* tokens,
                                       int32_t n_tok, int32_t overwrite) {
  return guard([&] {
    need(st && rec, "null argument");
    store_import(st->s, *rec, tokens, n_tok, overwrite != 0);
  });
}

FRAG_API frag_status frag_store_register_prefix(frag_store* st, const frag_chunk_id* sys_id, const frag_chunk_id* path,
                                                int32_t n) {
  return guard([&] {
    need(st, "null store");
    store_register_prefix(st->s, sys_id, path, n);
  });
}

FRAG_API frag_status frag_store_match(frag_store* st, const frag_chunk_id* sys_id, const frag_chunk_id* context,
                                      int32_t n, frag_match* out, int32_t* n_out) {
  return guard([&] {
    need(st && out && n_out, "null argument");
    *n_out = store_match(st->s, sys_id, context, n, out);
  });
}

FRAG_API int64_t frag_store_count(const frag_store* st) {
  if (!st) return -1;
  std::shared_lock<std::shared_mutex> g(st->s->mu);
  return (int64_t)st->s->recs.size();
}

FRAG_API uint64_t frag_store_bytes_used(const frag_store* st) {
  if (!st) return 0;
  std::shared_lock<std::shared_mutex> g(st->s->mu);
  return st->s->used;
}

FRAG_API frag_status frag_preprocess_isolated(frag_engine* eng, frag_store* st, const int32_t* sys, int32_t n_sys,
                                              const int32_t* tokens, int32_t n_tok, int32_t overwrite,
                                              frag_chunk_id* id_out) {
  return guard([&] {
    need(eng && st && tokens, "null argument");
    need(n_sys == 0 || sys, "null system prompt");
    preprocess_isolated(eng->e, st->s, sys, n_sys, tokens, n_tok, overwrite != 0, id_out);
  });
}

// ---------------------------------------------------------------- results
FRAG_API frag_status frag_preprocess_fused(frag_engine* eng, frag_store* src, frag_store* dst, const int32_t* sys,
                                          int32_t n_sys, const int32_t* tokens, int32_t n_tok,
                                          const frag_chunk_id* neighbors, int32_t n_neighbors, int32_t budget,
                                          int32_t overwrite, frag_chunk_id* id_out) {
  return guard([&] {
    need(eng && src && dst && tokens, "null argument");
    need(n_sys == 0 || sys, "null system prompt");
    preprocess_fused(eng->e, src->s, dst->s, sys, n_sys, tokens, n_tok, neighbors, n_neighbors, budget,
                     overwrite != 0, id_out);
  });
}

FRAG_API frag_status frag_result_create(frag_engine* eng, int32_t max_tokens, frag_result** out) {
  return guard([&] {
    need(eng && out, "null argument");
    auto* r = new Result();
    try {
      result_init(r, eng->e, max_tokens);
    } catch (...) {
      delete r;
      throw;
    }
    *out = new frag_result{r};
  });
}

FRAG_API frag_status frag_result_free(frag_result* res) {
  return guard([&] {
    if (!res) return;
    {
      DeviceGuard dg(res->r->eng->device);
      cudaDeviceSynchronize();
      delete res->r;
    }
    delete res;
  });
}

FRAG_API frag_status frag_reprocess(frag_engine* eng, frag_store* st, const int32_t* sys, int32_t n_sys,
                                    const int32_t* question, int32_t n_q, const frag_chunk_id* chunk_ids,
                                    int32_t n_chunks, float recompute_ratio, const frag_reprocess_opts* opts,
                                    void* stream, frag_result* res) {
  return guard([&] {
    need(eng && st && res && question, "null argument");
    need(n_sys == 0 || sys, "null system prompt");
    reprocess(eng->e, st->s, sys, n_sys, question, n_q, false, chunk_ids, n_chunks, recompute_ratio, opts,
              static_cast<cudaStream_t>(stream), res->r);
  });
}

FRAG_API frag_status frag_reprocess_dev(frag_engine* eng, frag_store* st, const int32_t* sys, int32_t n_sys,
                                        const int32_t* question_dev, int32_t n_q, const frag_chunk_id* chunk_ids,
                                        int32_t n_chunks, float recompute_ratio, const frag_reprocess_opts* opts,
                                        void* stream, frag_result* res) {
  return guard([&] {
    need(eng && st && res && question_dev, "null argument");
    need(n_sys == 0 || sys, "null system prompt");
    reprocess(eng->e, st->s, sys, n_sys, question_dev, n_q, true, chunk_ids, n_chunks, recompute_ratio, opts,
              static_cast<cudaStream_t>(stream), res->r);
  });
}

FRAG_API frag_status frag_full_prefill(frag_engine* eng, const int32_t* sys, int32_t n_sys, const int32_t* tokens,
                                       int32_t n_tok, const frag_reprocess_opts* opts, void* stream,
                                       frag_result* res) {
  return guard([&] {
    need(eng && res && tokens, "null argument");
    need(n_sys == 0 || sys, "null system prompt");
    full_prefill(eng->e, sys, n_sys, tokens, n_tok, opts, static_cast<cudaStream_t>(stream), res->r);
  });
}

FRAG_API frag_status frag_reprocess_batch(frag_engine* eng, frag_store* st, const frag_request* reqs, int32_t n_req,
                                          int32_t slot_tokens, const frag_reprocess_opts* opts, void* stream,
                                          frag_result* res) {
  return guard([&] {
    need(eng && st && res && reqs, "null argument");
    reprocess_batch(eng->e, st->s, reqs, n_req, slot_tokens, opts, static_cast<cudaStream_t>(stream), res->r);
  });
}

FRAG_API int32_t frag_result_batch_crit(const frag_result* res, int32_t b, int32_t* host_out, int32_t cap) {
  if (!res || b < 0 || b >= (int32_t)res->r->batch.size()) return -1;
  const auto& c = res->r->batch[b].crit;
  if (host_out)
    for (int32_t i = 0; i < (int32_t)c.size() && i < cap; ++i) host_out[i] = c[i];
  return (int32_t)c.size();
}

FRAG_API frag_status frag_kv_deviation(frag_engine* eng, frag_store* st, const int32_t* sys, int32_t n_sys,
                                       const frag_chunk_id* chunk_ids, int32_t n_chunks, int32_t n_layers,
                                       void* stream, frag_result* res, float* dev_host) {
  return guard([&] {
    need(eng && st && res && dev_host, "null argument");
    need(n_sys == 0 || sys, "null system prompt");
    kv_deviation(eng->e, st->s, sys, n_sys, chunk_ids, n_chunks, n_layers, static_cast<cudaStream_t>(stream), res->r,
                 dev_host);
  });
}

FRAG_API frag_status frag_decode(frag_engine* eng, frag_result* res, int32_t max_new_tokens, void* stream,
                                 int32_t* tokens_out) {
  return guard([&] {
    need(eng && res && tokens_out, "null argument");
    decode(eng->e, res->r, max_new_tokens, static_cast<cudaStream_t>(stream), tokens_out);
  });
}

FRAG_API frag_status frag_result_sync(frag_result* res) {
  return guard([&] {
    need(res, "null result");
    DeviceGuard dg(res->r->eng->device);
    check_cuda(cudaStreamSynchronize(res->r->last_stream), "sync");
  });
}

FRAG_API frag_status frag_result_fused_kv(const frag_result* res, const void** k_dev, const void** v_dev,
                                          int32_t* n_tokens) {
  return guard([&] {
    need(res, "null result");
    if (k_dev) *k_dev = res->r->k_fused.p;
    if (v_dev) {
      // shared V pages: the request's V view is assembled from its records and
      // exclusive slots on demand (stream-ordered after the request, synchronous)
      Result* r = res->r;
      DeviceGuard dg(r->eng->device);
      std::lock_guard<std::recursive_mutex> gpu_lock(device_mutex(r->eng->device));
      materialize_v(r, r->last_stream);
      *v_dev = r->v_fused.p;
    }
    if (n_tokens) *n_tokens = res->r->T;
  });
}

FRAG_API frag_status frag_result_logits(const frag_result* res, const float** logits, int32_t* rows,
                                        int32_t* vocab, int32_t on_device) {
  return guard([&] {
    need(res && logits, "null argument");
    const Result* r = res->r;
    if (on_device) {
      *logits = r->logits.as<float>();
    } else {
      need(!r->logits_on_device, "logits were kept on the device for this request");
      *logits = r->logits_host.as<float>();
    }
    if (rows) *rows = r->logit_rows;
    if (vocab) *vocab = r->eng->cfg.vocab;
  });
}

FRAG_API int32_t frag_result_crit(const frag_result* res, int32_t* host_out, int32_t cap) {
  if (!res) return -1;
  const Result* r = res->r;
  if (r->nq == 0) return 0;  // full prefill: no selection
  if (r->rows_per_seq > 0) return -1;  // batched: frag_result_batch_crit per request
  const int k = r->k_sel;
  if (host_out && cap > 0) {
    const int n = k < cap ? k : cap;
    DeviceGuard dg(r->eng->device);
    if (cudaMemcpy(host_out, r->plan_rows.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    for (int i = 0; i < n; ++i) host_out[i] += 1;  // rows -> 1-based positions
  }
  return k;
}

FRAG_API frag_status frag_result_timing(const frag_result* res, frag_timing* out) {
  return guard([&] {
    need(res && out, "null argument");
    *out = res->r->timing;  // stage fields are 0 unless the last call asked for timing
    if (!res->r->timing_valid) {
      const float hp = out->host_prep_ms;
      *out = frag_timing{};
      out->host_prep_ms = hp;
    }
  });
}

FRAG_API frag_status frag_result_debug(const frag_result* res, const float** q_final_dev, const float** scores_dev,
                                       int32_t* n_q, int32_t* n_chunk_tokens) {
  return guard([&] {
    need(res, "null result");
    if (q_final_dev) *q_final_dev = res->r->q_final.as<float>();
    if (scores_dev) *scores_dev = res->r->scores.as<float>();
    if (n_q) *n_q = res->r->nq;
    if (n_chunk_tokens) *n_chunk_tokens = res->r->N;
  });
}

// ---------------------------------------------------------------- kernels
FRAG_API frag_status frag_kernel_gemm(const void* a, const void* b, void* c, int32_t M, int32_t N, int32_t K,
                                      int32_t epi, int32_t force_bn, void* stream) {
  return guard([&] {
    need(a && b && c, "null argument");
    need(M >= 0 && N > 0 && K > 0, "bad shape");
    fragk::EpiParams ep;
    ep.ldo = N;
    fragk::EpiKind kind;
    if (epi == 0) {
      kind = fragk::EPI_STORE_BF16;
      ep.out_bf16 = static_cast<bf16*>(c);
    } else if (epi == 1) {
      kind = fragk::EPI_STORE_F32;
      ep.out_f32 = static_cast<float*>(c);
    } else if (epi == 2) {
      kind = fragk::EPI_RESID;
      ep.resid = static_cast<float*>(c);
    } else if (epi == 3) {
      kind = fragk::EPI_SWIGLU;
      ep.out_bf16 = static_cast<bf16*>(c);
      ep.ldo = N / 2;
    } else {
      fail(FRAG_E_CONTRACT, "unknown epilogue");
    }
    // split-K workspace for the small-M path (process-wide; this entry point is
    // for kernel-level tests and is serialised by the mutex)
    static std::mutex ws_mu;
    static DevBuf ws, cnt;
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    std::lock_guard<std::recursive_mutex> gd(fragimpl::device_mutex(dev));  // co-residency (engine.h)
    std::lock_guard<std::mutex> g(ws_mu);
    if (!ws.p) {
      ws.alloc((size_t)32 << 20);
      cnt.alloc(16384 * sizeof(int));
      check_cuda(cudaMemset(cnt.p, 0, cnt.bytes), "counter init");
    }
    ep.ws = ws.as<float>();
    ep.ws_bytes = ws.bytes;
    ep.counters = cnt.as<int>();
    ep.counters_cap = (int)(cnt.bytes / sizeof(int));
    const int n = fragk::gemm_bf16_tc(static_cast<const bf16*>(a), static_cast<const bf16*>(b), M, N, K, kind, ep,
                                      static_cast<cudaStream_t>(stream), force_bn);
    // flag 0x80000 (tuning tools): no synchronise, so back-to-back launches can
    // be timed; the caller keeps them on one stream
    if (!(force_bn & 0x80000)) {
      check_cuda(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "gemm");
      if (fragk::fault_take(dev)) {
        check_cuda(cudaMemset(cnt.p, 0, cnt.bytes), "counter re-arm");
        check_cuda(cudaDeviceSynchronize(), "counter re-arm");
        fail(FRAG_E_CUDA, "gemm: the persistent grid was not co-resident (inter-CTA wait limit exceeded)");
      }
    }
    if (n < 0) fail(FRAG_E_CONTRACT, "unsupported GEMM shape (K % 64, N % 64 and N % BN required)");
    g_launches += n;
    check_cuda(cudaPeekAtLastError(), "gemm launch");
  });
}

FRAG_API frag_status frag_kernel_rope_shift(const void* k_src, void* k_dst, int32_t L, int32_t n_tok, int32_t Hkv,
                                            int32_t dh, int32_t native_start, int32_t target_start,
                                            double rope_base, void* stream) {
  return guard([&] {
    need(k_src && k_dst, "null argument");
    need(L > 0 && n_tok > 0 && Hkv > 0 && (dh % 8) == 0, "bad shape");
    auto s = static_cast<cudaStream_t>(stream);
    const int delta = target_start - native_start;
    const int half = dh / 2;
    std::vector<float2> tab(half);
    for (int i = 0; i < half; ++i) {
      const double th = std::pow(rope_base, -2.0 * (double)(i + 1) / (double)dh);
      const double a = (double)delta * th;
      tab[i] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
    DevBuf dtab, ddesc, vtmp;
    dtab.alloc(half * sizeof(float2));
    ddesc.alloc(sizeof(fragk::StitchChunk));
    vtmp.alloc((size_t)L * n_tok * Hkv * dh * sizeof(bf16));
    fragk::StitchChunk c{static_cast<const bf16*>(k_src), static_cast<const bf16*>(k_src), n_tok, 0,
                         delta == 0 ? -1 : 0};
    check_cuda(cudaMemcpy(dtab.p, tab.data(), half * sizeof(float2), cudaMemcpyHostToDevice), "tab");
    check_cuda(cudaMemcpy(ddesc.p, &c, sizeof(c), cudaMemcpyHostToDevice), "desc");
    if (fragk::rope_shift_assemble(ddesc.as<fragk::StitchChunk>(), 1, n_tok, dtab.as<float2>(),
                                   static_cast<bf16*>(k_dst), vtmp.as<bf16>(), L, n_tok, Hkv, dh, s) < 0)
      fail(FRAG_E_CONTRACT, "kernel launch rejected the shape");
    g_launches += 1;
    check_cuda(cudaStreamSynchronize(s), "rope_shift");
  });
}

FRAG_API frag_status frag_kernel_qg_select(const float* q, const void* k, int32_t nq, int32_t Hq, int32_t Hkv,
                                           int32_t dh, int32_t n_keys, int32_t k_sel, int32_t raw,
                                           float* scores_dev, int32_t* sel_dev, void* stream) {
  return guard([&] {
    need(q && k && scores_dev && sel_dev, "null argument");
    need(nq > 0 && Hq > 0 && Hkv > 0 && Hq % Hkv == 0 && n_keys > 0, "bad shape");
    need(k_sel >= 0 && k_sel <= n_keys, "k out of range");
    auto s = static_cast<cudaStream_t>(stream);
    const int nblk = (n_keys + 31) / 32;
    DevBuf pms, rms, tok, ptok, col;
    pms.alloc((size_t)nblk * nq * Hq * sizeof(float2));
    col.alloc(fragk::score_col_part_elems(nq, Hq, Hkv, n_keys) * sizeof(float));
    DevBuf qsp;
    qsp.alloc(fragk::score_q_split_elems(nq, Hq, Hkv, dh) * sizeof(bf16));
    rms.alloc((size_t)nq * Hq * sizeof(float2));
    tok.alloc((size_t)n_keys * sizeof(int));
    ptok.alloc((size_t)(k_sel + 1) * sizeof(int));
    check_cuda(cudaMemset(tok.p, 0, (size_t)n_keys * sizeof(int)), "memset");
    fragk::ScoreArgs a{};
    a.q = q;
    a.k = static_cast<const bf16*>(k);
    a.nq = nq;
    a.Hq = Hq;
    a.Hkv = Hkv;
    a.dh = dh;
    a.key_row0 = 0;
    a.n_keys = n_keys;
    a.scale = 1.0f / std::sqrt((float)dh);
    a.part_ms = pms.as<float2>();
    a.row_ms = rms.as<float2>();
    a.scores = scores_dev;
    a.raw = raw;
    a.col_part = col.as<float>();
    a.q_split = qsp.as<bf16>();
    const int n1 = fragk::qg_score(a, s);
    if (n1 < 0) fail(FRAG_E_CONTRACT, "unsupported head_dim");
    fragk::topk_plan(scores_dev, n_keys, k_sel, 0, tok.as<int>(), tok.as<int>(), 0, 0, sel_dev, ptok.as<int>(), s);
    g_launches += n1 + 1;
    check_cuda(cudaStreamSynchronize(s), "qg_select");
  });
}

FRAG_API frag_status frag_kernel_attention(const void* q, const void* k, const void* v, const int32_t* rows,
                                           void* out, int32_t M, int32_t T, int32_t Hq, int32_t Hkv, int32_t dh,
                                           int32_t split_keys, void* stream) {
  return guard([&] {
    need(q && k && v && rows && out, "null argument");
    need(M > 0 && T > 0 && Hq % Hkv == 0, "bad shape");
    auto s = static_cast<cudaStream_t>(stream);
    fragk::AttnArgs a{};
    a.q = static_cast<const bf16*>(q);
    a.k = static_cast<const bf16*>(k);
    a.v = static_cast<const bf16*>(v);
    a.rows = rows;
    a.out = static_cast<bf16*>(out);
    a.M = M;
    a.T = T;
    a.Hq = Hq;
    a.Hkv = Hkv;
    a.dh = dh;
    a.scale = 1.0f / std::sqrt((float)dh);
    DevBuf po, pl;
    if (split_keys > 0) {
      need(split_keys % 64 == 0, "split_keys must be a multiple of 64");
      a.split_keys = split_keys;
      a.n_splits = (T + split_keys - 1) / split_keys;
      po.alloc((size_t)a.n_splits * M * Hq * dh * sizeof(float));
      pl.alloc((size_t)a.n_splits * M * Hq * sizeof(float));
      a.part_o = po.as<float>();
      a.part_lse = pl.as<float>();
    }
    const int n = fragk::sparse_q_attention(a, s);
    if (n < 0) fail(FRAG_E_CONTRACT, "unsupported attention shape");
    g_launches += n;
    check_cuda(cudaStreamSynchronize(s), "attention");
  });
}

}  // extern "C"
