// HBM-resident chunk-KV store: ChunkKVRecord, put_record
// (SPEC.md:265-273), fetch, reader/writer locking with pin
// counts. Records live in device memory of the store's GPU; the
// host keeps the index, heat metadata and a copy of each record's token ids.
// FKVC record files + the DISK -> GPU loader are
// at the end; tier eviction policy is out of scope (SURVEY.md §2 kv_store row).
#include <unistd.h>

#include <cstdio>
#include <cstring>
#include <memory>

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

// Insert an uploaded record under the writer lock: single copy per chunk id
// (SPEC.md:269), pinned records are never replaced, GPU-tier
// capacity accounting.
void store_insert(Store* st, std::unique_ptr<Record> rec, bool overwrite) {
  std::unique_lock<std::shared_mutex> g(st->mu);
  const ChunkKey key = key_of(rec->id);
  auto it = st->recs.find(key);
  size_t freed = 0;
  if (it != st->recs.end()) {
    if (!overwrite) fail(FRAG_E_STORE, "duplicate chunk record without overwrite (SPEC.md:269)");
    if (it->second->pins > 0) fail(FRAG_E_STORE, "cannot overwrite a pinned record (SPEC.md:320)");
    if (it->second->exported) fail(FRAG_E_STORE, "cannot overwrite a record exported to peer GPUs");
    freed = it->second->tier == FRAG_TIER_PEER ? 0 : it->second->bytes;
  }
  // peer views occupy no local HBM
  const size_t bytes = rec->tier == FRAG_TIER_PEER ? 0 : rec->bytes;
  if (st->capacity && st->used - freed + bytes > st->capacity)
    fail(FRAG_E_STORE, "GPU tier capacity exhausted (tiering/eviction out of scope in this build)");
  if (it != st->recs.end()) {
    st->used -= freed;
    it->second = std::shared_ptr<Record>(std::move(rec));
  } else {
    st->recs.emplace(key, std::shared_ptr<Record>(std::move(rec)));
  }
  st->used += bytes;
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
  const ChunkKey key = key_of(id);
  {
    std::shared_lock<std::shared_mutex> g(st->mu);  // early duplicate check (re-checked at insert)
    if (!overwrite && st->recs.count(key)) fail(FRAG_E_STORE, "duplicate chunk record without overwrite (SPEC.md:269)");
  }
  // upload outside the store lock: readers (reprocess) keep going meanwhile
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
  store_insert(st, std::move(rec), overwrite);
}

namespace {
// fetch from this store's own index only (heat++, pin); null on a miss
Record* fetch_local(Store* st, const ChunkKey& key) {
  std::unique_lock<std::shared_mutex> g(st->mu);  // heat/pin are mutated
  auto it = st->recs.find(key);
  if (it == st->recs.end()) return nullptr;
  Record* r = it->second.get();
  r->heat += 1;
  r->last_access = ++st->tick;
  r->pins += 1;
  return r;
}
bool release_local(Store* st, const ChunkKey& key) {
  std::unique_lock<std::shared_mutex> g(st->mu);
  auto it = st->recs.find(key);
  if (it == st->recs.end()) return false;
  if (it->second->pins > 0) it->second->pins -= 1;
  return true;
}
}  // namespace

// A miss in this store falls through to the attached same-process peers (the
// owning store keeps heat and pins); cross-process records were imported into
// the local index as FRAG_TIER_PEER views and hit locally.
Record* store_try_fetch(Store* st, const frag_chunk_id& id) {
  const ChunkKey key = key_of(id);
  if (Record* r = fetch_local(st, key)) return r;
  std::vector<Store*> peers;
  {
    std::shared_lock<std::shared_mutex> g(st->mu);
    peers = st->peers;
  }
  for (Store* p : peers)
    if (Record* r = fetch_local(p, key)) return r;
  return nullptr;
}

Record* store_fetch(Store* st, const frag_chunk_id& id) {
  if (Record* r = store_try_fetch(st, id)) return r;
  fail(FRAG_E_STORE, "missing chunk record (SPEC.md:287)");
}

void store_release(Store* st, const frag_chunk_id& id) {
  const ChunkKey key = key_of(id);
  if (release_local(st, key)) return;
  std::vector<Store*> peers;
  {
    std::shared_lock<std::shared_mutex> g(st->mu);
    peers = st->peers;
  }
  for (Store* p : peers)
    if (release_local(p, key)) return;
  fail(FRAG_E_STORE, "missing chunk record");
}

Record::~Record() {
  if (ipc_mapped && kv.p) {
    cudaIpcCloseMemHandle(kv.p);  // a mapping of the owner's pages: never cudaFree'd here
    kv.p = nullptr;
    kv.bytes = 0;
  }
}

// ---------------------------------------------------------------- alternative_path_match
// PrefixKey: two splitmix64-mixed lanes seeded by the
// system-prompt id, folded over the ordered chunk ids, finalised with the
// path length.
ChunkKey prefix_key(const frag_chunk_id* sys_id, const frag_chunk_id* path, int n) {
  ChunkKey s{0x6a09e667f3bcc908ULL, 0xbb67ae8584caa73bULL};
  if (sys_id) {
    const ChunkKey k = key_of(*sys_id);
    s.a ^= k.a;
    s.b ^= k.b;
  }
  uint64_t a = mix64(s.a), b = mix64(s.b + 0x9e3779b97f4a7c15ULL);
  for (int i = 0; i < n; ++i) {
    const ChunkKey c = key_of(path[i]);
    a = mix64(a ^ mix64(c.a + 0x3c6ef372fe94f82bULL * (uint64_t)(i + 1)));
    b = mix64(b + mix64(c.b ^ 0xa54ff53a5f1d36f1ULL) + (uint64_t)i);
  }
  return ChunkKey{mix64(a ^ (uint64_t)n), mix64(b + (uint64_t)n * 0x9e3779b97f4a7c15ULL)};
}

void store_register_prefix(Store* st, const frag_chunk_id* sys_id, const frag_chunk_id* path, int n) {
  if (n < 1 || !path) fail(FRAG_E_CONTRACT, "a cached path needs at least one chunk");
  const ChunkKey pk = prefix_key(sys_id, path, n);
  std::unique_lock<std::shared_mutex> g(st->mu);
  st->prefix_index[pk] = key_of(path[n - 1]);
}

// Progressive backtracking (design decision SPEC.md:317): for
// context chunk i try the full preceding path, then drop the EARLIEST
// remaining preceding chunk, down to the chunk alone; a hit must name chunk i
// and its record must still exist (here or in an attached peer).
int store_match(Store* st, const frag_chunk_id* sys_id, const frag_chunk_id* ctx, int n, frag_match* out) {
  if (n < 1 || !ctx) fail(FRAG_E_CONTRACT, "context must be non-empty (SPEC.md:276)");
  std::vector<Store*> stores{st};
  {
    std::shared_lock<std::shared_mutex> g(st->mu);
    stores.insert(stores.end(), st->peers.begin(), st->peers.end());
  }
  auto has_record = [&](const ChunkKey& k) {
    for (Store* s : stores) {
      std::shared_lock<std::shared_mutex> g(s->mu);
      if (s->recs.count(k)) return true;
    }
    return false;
  };
  int m = 0;
  for (int i = 0; i < n; ++i) {
    const ChunkKey ck = key_of(ctx[i]);
    if (!has_record(ck)) continue;  // uncached: absent from the result
    int hit = -1;
    for (int start = 0; start <= i && hit < 0; ++start) {
      const ChunkKey pk = prefix_key(sys_id, ctx + start, i - start + 1);
      std::shared_lock<std::shared_mutex> g(st->mu);
      auto it = st->prefix_index.find(pk);
      if (it != st->prefix_index.end() && it->second == ck) hit = start;
    }
    out[m].id = ctx[i];
    out[m].position = i;
    out[m].path_start = hit >= 0 ? hit : i;
    out[m].matched_via = hit == 0 ? FRAG_MATCH_PREFIX : FRAG_MATCH_ALT_PATH;
    ++m;
  }
  return m;
}

// ---------------------------------------------------------------- partitioned store
int32_t chunk_owner(const frag_chunk_id& id, int32_t n) {
  if (n < 1) fail(FRAG_E_CONTRACT, "n_owners must be >= 1");
  uint64_t a = 0;
  for (int i = 7; i >= 0; --i) a = (a << 8) | id.bytes[i];
  return (int32_t)(a % (uint64_t)n);
}

void store_attach_peer(Store* local, Store* remote) {
  if (!local || !remote) fail(FRAG_E_CONTRACT, "null store");
  if (local == remote) fail(FRAG_E_CONTRACT, "a store cannot be its own peer");
  const auto &a = local->cfg, &b = remote->cfg;
  if (a.layers != b.layers || a.n_kv_heads != b.n_kv_heads || a.head_dim != b.head_dim || a.vocab != b.vocab)
    fail(FRAG_E_CONTRACT, "peer store has a different record layout");
  if (local->device != remote->device) {
    DeviceGuard dg(local->device);
    int ok = 0;
    check_cuda(cudaDeviceCanAccessPeer(&ok, local->device, remote->device), "cudaDeviceCanAccessPeer");
    if (!ok) fail(FRAG_E_CUDA, "no peer access between device " + std::to_string(local->device) + " and " +
                                   std::to_string(remote->device));
    const cudaError_t e = cudaDeviceEnablePeerAccess(remote->device, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled)
      cudaGetLastError();
    else
      check_cuda(e, "cudaDeviceEnablePeerAccess");
  }
  std::unique_lock<std::shared_mutex> g(local->mu);
  for (Store* p : local->peers)
    if (p == remote) return;
  local->peers.push_back(remote);
}

namespace {
// physical identity of a device (PCI domain / bus / device), independent of
// each process's device numbering (CUDA_VISIBLE_DEVICES may differ per rank)
int32_t pci_key(int dev) {
  int dom = 0, bus = 0, slot = 0;
  check_cuda(cudaDeviceGetAttribute(&dom, cudaDevAttrPciDomainId, dev), "pci domain");
  check_cuda(cudaDeviceGetAttribute(&bus, cudaDevAttrPciBusId, dev), "pci bus");
  check_cuda(cudaDeviceGetAttribute(&slot, cudaDevAttrPciDeviceId, dev), "pci device");
  return (int32_t)(((uint32_t)(dom & 0xFFFF) << 16) | ((uint32_t)(bus & 0xFF) << 8) | (uint32_t)(slot & 0xFF));
}
}  // namespace

void store_export(Store* st, const frag_chunk_id& id, frag_peer_record* out) {
  if (!out) fail(FRAG_E_CONTRACT, "null output");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  std::unique_lock<std::shared_mutex> g(st->mu);
  auto it = st->recs.find(key_of(id));
  if (it == st->recs.end()) fail(FRAG_E_STORE, "missing chunk record (SPEC.md:287)");
  Record* r = it->second.get();
  if (r->tier == FRAG_TIER_PEER) fail(FRAG_E_CONTRACT, "only the owning store can export a record");
  DeviceGuard dg(st->device);
  cudaIpcMemHandle_t h;
  check_cuda(cudaIpcGetMemHandle(&h, r->kv.p), "cudaIpcGetMemHandle");
  std::memset(out, 0, sizeof(*out));
  out->id = r->id;
  out->n_tok = r->n_tok;
  out->native_start = r->native_start;
  out->variant = r->variant;
  out->owner_device = st->device;
  out->layers = st->cfg.layers;
  out->n_kv_heads = st->cfg.n_kv_heads;
  out->head_dim = st->cfg.head_dim;
  out->kv_bytes = r->kv.bytes;
  out->owner_pid = (uint64_t)getpid();
  out->owner_pci = pci_key(st->device);  // owner GPU's PCI id (distinct-device imports)
  std::memcpy(out->ipc_handle, &h, sizeof(h));
  r->exported = true;
}

void store_import(Store* st, const frag_peer_record& pr, const int32_t* tokens, int n_tok, bool overwrite) {
  const auto& c = st->cfg;
  if (pr.layers != c.layers || pr.n_kv_heads != c.n_kv_heads || pr.head_dim != c.head_dim)
    fail(FRAG_E_CONTRACT, "peer record has a different record layout");
  if (pr.n_tok < 1 || pr.n_tok != n_tok) fail(FRAG_E_CONTRACT, "token count does not match the peer record");
  if (pr.kv_bytes != st->record_bytes(n_tok)) fail(FRAG_E_CONTRACT, "peer record size does not match its shape");
  if (pr.native_start < 1) fail(FRAG_E_CONTRACT, "native_start must be >= 1 (SPEC.md:257)");
  if (pr.variant != FRAG_VARIANT_ISOLATED && pr.variant != FRAG_VARIANT_FUSED) fail(FRAG_E_CONTRACT, "unknown variant");
  if (pr.owner_pid == (uint64_t)getpid())
    fail(FRAG_E_CONTRACT, "record was exported by this process: use frag_store_attach_peer");
  if (!tokens) fail(FRAG_E_CONTRACT, "null tokens");
  for (int i = 0; i < n_tok; ++i)
    if (tokens[i] < 0 || tokens[i] >= c.vocab) fail(FRAG_E_CONTRACT, "record token out of vocabulary");
  {
    std::shared_lock<std::shared_mutex> g(st->mu);
    if (!overwrite && st->recs.count(key_of(pr.id)))
      fail(FRAG_E_STORE, "duplicate chunk record without overwrite (SPEC.md:269)");
  }
  DeviceGuard dg(st->device);
  if (pr.owner_pci != 0 && pr.owner_pci != pci_key(st->device)) {
    // the owner is another GPU: K1 reads its pages over NVLink -- it must be
    // visible to this process and peer-accessible from this store's device
    int n_dev = 0, owner = -1;
    check_cuda(cudaGetDeviceCount(&n_dev), "cudaGetDeviceCount");
    for (int d = 0; d < n_dev && owner < 0; ++d)
      if (pci_key(d) == pr.owner_pci) owner = d;
    if (owner < 0) fail(FRAG_E_CUDA, "peer record's GPU is not visible to this process (CUDA_VISIBLE_DEVICES)");
    int ok = 0;
    check_cuda(cudaDeviceCanAccessPeer(&ok, st->device, owner), "cudaDeviceCanAccessPeer");
    if (!ok)
      fail(FRAG_E_CUDA, "no peer access from device " + std::to_string(st->device) + " to the owner (device " +
                            std::to_string(owner) + ")");
  }
  auto rec = std::make_unique<Record>();
  rec->id = pr.id;
  rec->n_tok = n_tok;
  rec->native_start = pr.native_start;
  rec->variant = pr.variant;
  rec->bytes = pr.kv_bytes;
  rec->tier = FRAG_TIER_PEER;
  rec->owner_device = pr.owner_device;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, pr.ipc_handle, sizeof(h));
  void* p = nullptr;
  check_cuda(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  rec->kv.p = p;
  rec->kv.bytes = pr.kv_bytes;
  rec->ipc_mapped = true;
  rec->tok.alloc(n_tok * sizeof(int32_t));  // token ids are local (K2 gathers their embeddings)
  rec->tok_host.assign(tokens, tokens + n_tok);
  check_cuda(cudaMemcpy(rec->tok.p, tokens, n_tok * sizeof(int32_t), cudaMemcpyHostToDevice), "peer record tokens");
  store_insert(st, std::move(rec), overwrite);
}

// ---------------------------------------------------------------- FKVC files
namespace {
constexpr uint32_t kFkvcVersion = 1;
constexpr size_t kFkvcHeader = 4 + 4 + 16 + 1 + 4 + 2 + 2 + 2 + 4;  // 39 bytes, packed little-endian

struct FileCloser {
  void operator()(FILE* f) const {
    if (f) std::fclose(f);
  }
};
using FilePtr = std::unique_ptr<FILE, FileCloser>;

template <class T>
void put_le(uint8_t*& p, T v) {
  for (size_t i = 0; i < sizeof(T); ++i) *p++ = (uint8_t)((uint64_t)v >> (8 * i));
}
template <class T>
T get_le(const uint8_t*& p) {
  uint64_t v = 0;
  for (size_t i = 0; i < sizeof(T); ++i) v |= (uint64_t)(*p++) << (8 * i);
  return (T)v;
}

void encode_header(const frag_fkvc_header& h, uint8_t* buf) {
  uint8_t* p = buf;
  std::memcpy(p, "FKVC", 4);
  p += 4;
  put_le<uint32_t>(p, kFkvcVersion);
  std::memcpy(p, h.id.bytes, 16);
  p += 16;
  put_le<uint8_t>(p, (uint8_t)h.variant);
  put_le<uint32_t>(p, (uint32_t)h.native_start);
  put_le<uint16_t>(p, (uint16_t)h.layers);
  put_le<uint16_t>(p, (uint16_t)h.heads);
  put_le<uint16_t>(p, (uint16_t)h.head_dim);
  put_le<uint32_t>(p, (uint32_t)h.tokens);
}

frag_fkvc_header read_header(FILE* f, const char* path) {
  uint8_t buf[kFkvcHeader];
  const size_t got = std::fread(buf, 1, kFkvcHeader, f);
  if (got >= 4 && std::memcmp(buf, "FKVC", 4) != 0) fail_format(FRAG_FORMAT_BAD_MAGIC, std::string("not an FKVC file: ") + path);
  if (got < kFkvcHeader) fail_format(FRAG_FORMAT_TRUNCATED, std::string("truncated FKVC header: ") + path);
  const uint8_t* p = buf + 4;
  const uint32_t ver = get_le<uint32_t>(p);
  if (ver != kFkvcVersion)
    fail_format(FRAG_FORMAT_BAD_VERSION, "FKVC version " + std::to_string(ver) + " (expected 1): " + path);
  frag_fkvc_header h{};
  std::memcpy(h.id.bytes, p, 16);
  p += 16;
  h.variant = get_le<uint8_t>(p);
  h.native_start = (int32_t)get_le<uint32_t>(p);
  h.layers = get_le<uint16_t>(p);
  h.heads = get_le<uint16_t>(p);
  h.head_dim = get_le<uint16_t>(p);
  h.tokens = (int32_t)get_le<uint32_t>(p);
  if (h.layers < 1 || h.heads < 1 || h.head_dim < 1 || h.tokens < 1 || h.native_start < 1 ||
      (h.variant != FRAG_VARIANT_ISOLATED && h.variant != FRAG_VARIANT_FUSED))
    fail_format(FRAG_FORMAT_MALFORMED, std::string("malformed FKVC header: ") + path);
  return h;
}

void read_exact(FILE* f, void* dst, size_t bytes, const char* path) {
  if (std::fread(dst, 1, bytes, f) != bytes)
    fail_format(FRAG_FORMAT_TRUNCATED, std::string("truncated FKVC payload: ") + path);
}

FilePtr open_or_fail(const char* path, const char* mode) {
  FilePtr f(std::fopen(path, mode));
  if (!f) fail_format(FRAG_FORMAT_IO, std::string("cannot open ") + path);
  return f;
}
}  // namespace

void fkvc_write(const char* path, const frag_fkvc_header& h, const float* k, const float* v) {
  if (h.layers < 1 || h.heads < 1 || h.head_dim < 1 || h.tokens < 1 || h.native_start < 1)
    fail(FRAG_E_CONTRACT, "invalid FKVC header fields");
  FilePtr f = open_or_fail(path, "wb");
  uint8_t buf[kFkvcHeader];
  encode_header(h, buf);
  bool ok = std::fwrite(buf, 1, kFkvcHeader, f.get()) == kFkvcHeader;
  const size_t per = (size_t)h.tokens * h.heads * h.head_dim;
  for (int l = 0; l < h.layers && ok; ++l) {
    ok = std::fwrite(k + (size_t)l * per, sizeof(float), per, f.get()) == per &&
         std::fwrite(v + (size_t)l * per, sizeof(float), per, f.get()) == per;
  }
  if (!ok || std::fflush(f.get()) != 0) fail_format(FRAG_FORMAT_IO, std::string("write failed: ") + path);
}

void fkvc_read(const char* path, frag_fkvc_header* h, float* k, float* v, size_t cap_floats) {
  FilePtr f = open_or_fail(path, "rb");
  *h = read_header(f.get(), path);
  if (!k && !v) return;
  const size_t per = (size_t)h->tokens * h->heads * h->head_dim;
  if (!k || !v || cap_floats < per * h->layers) fail(FRAG_E_CONTRACT, "output buffers too small for the FKVC record");
  for (int l = 0; l < h->layers; ++l) {
    read_exact(f.get(), k + (size_t)l * per, per * sizeof(float), path);
    read_exact(f.get(), v + (size_t)l * per, per * sizeof(float), path);
  }
}

void store_save(Store* st, const frag_chunk_id& id, const char* path) {
  const auto& c = st->cfg;
  DeviceGuard dg(st->device);
  Record* r = nullptr;
  {  // pin while it is read (saving is not an access: heat unchanged)
    std::unique_lock<std::shared_mutex> g(st->mu);
    auto it = st->recs.find(key_of(id));
    if (it == st->recs.end()) fail(FRAG_E_STORE, "missing chunk record (SPEC.md:287)");
    r = it->second.get();
    r->pins += 1;
  }
  struct Unpin {
    Store* st;
    frag_chunk_id id;
    ~Unpin() {
      try {
        store_release(st, id);
      } catch (...) {
      }
    }
  } unpin{st, id};
  const size_t per = (size_t)r->n_tok * c.n_kv_heads * c.head_dim;
  std::vector<uint16_t> kb(per * c.layers), vb(per * c.layers);
  check_cuda(cudaMemcpy(kb.data(), r->k(), kb.size() * 2, cudaMemcpyDeviceToHost), "record K D2H");
  check_cuda(cudaMemcpy(vb.data(), r->v(), vb.size() * 2, cudaMemcpyDeviceToHost), "record V D2H");
  std::vector<float> kf(kb.size()), vf(vb.size());
  for (size_t i = 0; i < kb.size(); ++i) {  // bf16 -> fp32 is exact
    uint32_t a = (uint32_t)kb[i] << 16, b = (uint32_t)vb[i] << 16;
    std::memcpy(&kf[i], &a, 4);
    std::memcpy(&vf[i], &b, 4);
  }
  frag_fkvc_header h{};
  h.id = r->id;
  h.variant = r->variant;
  h.native_start = r->native_start;
  h.layers = c.layers;
  h.heads = c.n_kv_heads;
  h.head_dim = c.head_dim;
  h.tokens = r->n_tok;
  fkvc_write(path, h, kf.data(), vf.data());
}

void store_load(Store* st, const char* path, const int32_t* tokens, int n_tok, bool overwrite, cudaStream_t s,
                frag_chunk_id* id_out) {
  const auto& c = st->cfg;
  FilePtr f = open_or_fail(path, "rb");
  const frag_fkvc_header h = read_header(f.get(), path);
  if (h.layers != c.layers || h.heads != c.n_kv_heads || h.head_dim != c.head_dim)
    fail_format(FRAG_FORMAT_MALFORMED, std::string("FKVC record shape does not match the store's model: ") + path);
  if (n_tok != h.tokens) fail(FRAG_E_CONTRACT, "token count differs from the FKVC record's");
  for (int i = 0; i < n_tok; ++i)
    if (tokens[i] < 0 || tokens[i] >= c.vocab) fail(FRAG_E_CONTRACT, "record token out of vocabulary");
  const ChunkKey key = key_of(h.id);
  {
    std::shared_lock<std::shared_mutex> g(st->mu);
    if (!overwrite && st->recs.count(key)) fail(FRAG_E_STORE, "duplicate chunk record without overwrite (SPEC.md:269)");
  }
  DeviceGuard dg(st->device);
  const size_t per = (size_t)n_tok * c.n_kv_heads * c.head_dim;  // floats of K (or V) per layer
  auto rec = std::make_unique<Record>();
  rec->id = h.id;
  rec->n_tok = n_tok;
  rec->native_start = h.native_start;
  rec->variant = h.variant;
  rec->bytes = st->record_bytes(n_tok);
  rec->kv.alloc(rec->bytes);
  rec->tok.alloc(n_tok * sizeof(int32_t));
  rec->tok_host.assign(tokens, tokens + n_tok);
  // ping-pong: read layer l+1 from the file while layer l is copied + converted
  PinnedBuf host[2];
  DevBuf dev[2];
  cudaEvent_t done[2] = {nullptr, nullptr};
  for (int b = 0; b < 2; ++b) {
    host[b].ensure(2 * per * sizeof(float));
    dev[b].alloc(2 * per * sizeof(float));
    check_cuda(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming), "event");
  }
  struct Events {
    cudaEvent_t* e;
    ~Events() {
      for (int b = 0; b < 2; ++b)
        if (e[b]) cudaEventDestroy(e[b]);
    }
  } ev_guard{done};
  bool in_flight[2] = {false, false};
  for (int l = 0; l < c.layers; ++l) {
    const int b = l & 1;
    if (in_flight[b]) check_cuda(cudaEventSynchronize(done[b]), "loader buffer");
    read_exact(f.get(), host[b].p, 2 * per * sizeof(float), path);  // K then V of layer l
    check_cuda(cudaMemcpyAsync(dev[b].p, host[b].p, 2 * per * sizeof(float), cudaMemcpyHostToDevice, s), "H2D");
    fragk::f32_to_bf16(dev[b].as<float>(), rec->k() + (size_t)l * per, per, s);
    fragk::f32_to_bf16(dev[b].as<float>() + per, rec->v() + (size_t)l * per, per, s);
    check_cuda(cudaEventRecord(done[b], s), "event record");
    in_flight[b] = true;
  }
  g_launches += 2 * (uint64_t)c.layers;
  check_cuda(cudaMemcpyAsync(rec->tok.p, tokens, n_tok * sizeof(int32_t), cudaMemcpyHostToDevice, s), "tokens");
  check_cuda(cudaStreamSynchronize(s), "record load");
  if (id_out) *id_out = h.id;
  store_insert(st, std::move(rec), overwrite);
}

}  // namespace fragimpl
