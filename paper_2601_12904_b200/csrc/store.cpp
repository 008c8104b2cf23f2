// HBM-resident chunk-KV store: ChunkKVRecord, put_record
// (SPEC.md:265-273), fetch, reader/writer locking with pin
// counts. Records live in device memory of the store's GPU; the
// host keeps the index, heat metadata and a copy of each record's token ids.
// Tiering (CPU/DISK), eviction and the FKVC file format are out of scope
// (SURVEY.md §2 kv_store row, §8(f) rank 2).
#include <cstring>

#include "engine.h"

namespace fragimpl {

ChunkKey key_of(const frag_chunk_id& id) {
  ChunkKey k;
  std::memcpy(&k.a, id.bytes, 8);
  std::memcpy(&k.b, id.bytes + 8, 8);
  return k;
}

namespace {
uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
}  // namespace

// hash_tokens (common.hpp:122; body not shipped by the reference): two
// independent splitmix64-mixed lanes over (index, token), finalised with the
// length. Only equality semantics are relied upon.
void hash_tokens(const int32_t* t, int n, uint64_t salt, frag_chunk_id* out) {
  uint64_t a = 0x243f6a8885a308d3ULL ^ salt;
  uint64_t b = 0x13198a2e03707344ULL ^ mix64(salt + 1);
  for (int i = 0; i < n; ++i) {
    const uint64_t u = (uint64_t)(uint32_t)t[i];
    a = mix64(a + 0x9e3779b97f4a7c15ULL * (u + 1) + (uint64_t)i);
    b = mix64(b ^ (u * 0xd1b54a32d192ed03ULL + 0x8cb92ba72f3d8dd7ULL * (uint64_t)(i + 1)));
  }
  a = mix64(a ^ (uint64_t)n);
  b = mix64(b + (uint64_t)n * 0x9e3779b97f4a7c15ULL);
  std::memcpy(out->bytes, &a, 8);
  std::memcpy(out->bytes + 8, &b, 8);
}

Store* store_create(const frag_model_cfg& cfg, int device, size_t cap) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    fail(FRAG_E_CUDA, "no CUDA device available");
  }
  if (device < 0 || device >= ndev) fail(FRAG_E_CONTRACT, "device ordinal out of range");
  auto* s = new Store();
  s->cfg = cfg;
  s->device = device;
  s->capacity = cap;
  return s;
}

void store_put(Store* st, const frag_chunk_id& id, const int32_t* tokens, int n_tok, int native_start, int variant,
               const void* k, const void* v, bool overwrite, size_t src_layer_pitch_elems, cudaStream_t s) {
  const auto& c = st->cfg;
  if (n_tok < 1) fail(FRAG_E_CONTRACT, "record must hold at least one token");
  if (native_start < 1) fail(FRAG_E_CONTRACT, "native_start must be >= 1 (SPEC.md:257)");
  if (variant != FRAG_VARIANT_ISOLATED && variant != FRAG_VARIANT_FUSED) fail(FRAG_E_CONTRACT, "unknown variant");
  if (!tokens || !k || !v) fail(FRAG_E_CONTRACT, "null record buffer");
  for (int i = 0; i < n_tok; ++i)
    if (tokens[i] < 0 || tokens[i] >= c.vocab) fail(FRAG_E_CONTRACT, "record token out of vocabulary");
  const size_t bytes = st->record_bytes(n_tok);
  DeviceGuard dg(st->device);
  std::unique_lock<std::shared_mutex> g(st->mu);
  const ChunkKey key = key_of(id);
  auto it = st->recs.find(key);
  size_t freed = 0;
  if (it != st->recs.end()) {
    if (!overwrite) fail(FRAG_E_STORE, "duplicate chunk record without overwrite (SPEC.md:269)");
    if (it->second->pins > 0) fail(FRAG_E_STORE, "cannot overwrite a pinned record (SPEC.md:320)");
    freed = it->second->bytes;
  }
  if (st->capacity && st->used - freed + bytes > st->capacity)
    fail(FRAG_E_STORE, "GPU tier capacity exhausted (tiering/eviction out of scope in this build)");
  auto rec = std::make_unique<Record>();
  rec->id = id;
  rec->n_tok = n_tok;
  rec->native_start = native_start;
  rec->variant = variant;
  rec->bytes = bytes;
  rec->kv.alloc(bytes);
  rec->tok.alloc(n_tok * sizeof(int32_t));
  rec->tok_host.assign(tokens, tokens + n_tok);
  const size_t kvc = (size_t)c.n_kv_heads * c.head_dim;
  const size_t w = (size_t)n_tok * kvc * sizeof(bf16);
  const size_t pitch = src_layer_pitch_elems ? src_layer_pitch_elems * sizeof(bf16) : w;
  check_cuda(cudaMemcpy2DAsync(rec->kv.p, w, k, pitch, w, c.layers, cudaMemcpyDefault, s), "record K");
  check_cuda(cudaMemcpy2DAsync(rec->kv.as<char>() + (size_t)c.layers * w, w, v, pitch, w, c.layers,
                               cudaMemcpyDefault, s),
             "record V");
  check_cuda(cudaMemcpyAsync(rec->tok.p, tokens, n_tok * sizeof(int32_t), cudaMemcpyDefault, s), "record tokens");
  check_cuda(cudaStreamSynchronize(s), "record upload");
  if (it != st->recs.end()) {
    st->used -= freed;
    it->second = std::move(rec);
  } else {
    st->recs.emplace(key, std::move(rec));
  }
  st->used += bytes;
}

Record* store_fetch(Store* st, const frag_chunk_id& id) {
  std::unique_lock<std::shared_mutex> g(st->mu);  // heat/pin are mutated
  auto it = st->recs.find(key_of(id));
  if (it == st->recs.end()) fail(FRAG_E_STORE, "missing chunk record (SPEC.md:287)");
  Record* r = it->second.get();
  r->heat += 1;
  r->last_access = ++st->tick;
  r->pins += 1;
  return r;
}

void store_release(Store* st, const frag_chunk_id& id) {
  std::unique_lock<std::shared_mutex> g(st->mu);
  auto it = st->recs.find(key_of(id));
  if (it == st->recs.end()) fail(FRAG_E_STORE, "missing chunk record");
  if (it->second->pins > 0) it->second->pins -= 1;
}

}  // namespace fragimpl
