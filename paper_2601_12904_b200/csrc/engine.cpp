// Host orchestration of the online reprocessing stage:
//   stitch_full_reuse (K1) -> question pass (last_layer_query_states)
//   -> select_query_guided (K9, K10) -> sparse prefill (K2..K8 per layer) -> lm_head (K11).
// The whole request is stream-ordered; the only host synchronisation is the
// final one that makes the first-token logits visible (the TTFT end).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>

#include <cstdlib>

#include "engine.h"

namespace fragimpl {

std::recursive_mutex& device_mutex(int device) {
  static std::recursive_mutex mu[64];
  return mu[(unsigned)device % 64u];
}

// Stream synchronisation at the end of a call + the co-residency check of its
// persistent grids (ptx.cuh spin_until_ge): a grid that abandoned an
// inter-CTA wait voids the call's results; its counters are re-armed here.
void sync_checked(Engine* e, Result* r, cudaStream_t s, const char* what) {
  check_cuda(cudaStreamSynchronize(s), what);
  if (!fragk::fault_take(e->device)) return;
  check_cuda(cudaDeviceSynchronize(), "co-residency fault drain");
  if (r && r->gemm_cnt.p) check_cuda(cudaMemset(r->gemm_cnt.p, 0, r->gemm_cnt.bytes), "counter re-arm");
  if (e->scratch && e->scratch.get() != r && e->scratch->gemm_cnt.p)
    check_cuda(cudaMemset(e->scratch->gemm_cnt.p, 0, e->scratch->gemm_cnt.bytes), "counter re-arm");
  check_cuda(cudaDeviceSynchronize(), "counter re-arm");
  fail(FRAG_E_CUDA, std::string(what) +
                        ": a persistent kernel grid was not co-resident (an inter-CTA wait exceeded "
                        "FRAG_SPIN_LIMIT_MS; another context holds SMs?) -- the call's results are void");
}


std::atomic<uint64_t> g_launches{0};
std::atomic<uint64_t> g_alloc_epoch{0};

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    if (e == cudaErrorMemoryAllocation) fail(FRAG_E_OOM, std::string(what) + ": " + cudaGetErrorString(e));
    fail(FRAG_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

void DevBuf::alloc(size_t n) {
  release();
  g_alloc_epoch++;  // invalidates captured request graphs
  if (n == 0) return;
  cudaError_t e = cudaMalloc(&p, n);
  if (e != cudaSuccess) {
    p = nullptr;
    cudaGetLastError();
    fail(FRAG_E_OOM, "cudaMalloc(" + std::to_string(n) + " bytes) failed: " + cudaGetErrorString(e));
  }
  bytes = n;
}
void DevBuf::ensure(size_t n) {
  if (n > bytes) alloc(n);
}
void PinnedBuf::ensure(size_t n) {
  if (n <= bytes) return;
  if (p) cudaFreeHost(p);
  p = nullptr;
  bytes = 0;
  check_cuda(cudaMallocHost(&p, n), "cudaMallocHost");
  g_alloc_epoch++;  // captured graphs may copy from/to pinned buffers
  bytes = n;
}

DeviceGuard::DeviceGuard(int dev) {
  cudaGetDevice(&prev);
  if (prev != dev) check_cuda(cudaSetDevice(dev), "cudaSetDevice");
}
DeviceGuard::~DeviceGuard() {
  int cur = -1;
  cudaGetDevice(&cur);
  if (prev >= 0 && cur != prev) cudaSetDevice(prev);
}

// ---------------------------------------------------------------- profiler
cudaEvent_t Profiler::get() {
  if (!pool.empty()) {
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  check_cuda(cudaEventCreate(&e), "cudaEventCreate");
  return e;
}
void Profiler::begin(cudaStream_t s, cudaEvent_t* a) {
  if (!on) return;
  *a = get();
  cudaEventRecord(*a, s);
}
void Profiler::end(cudaStream_t s, cudaEvent_t a, int klass, double fl, double by, int nl) {
  if (!on) return;
  cudaEvent_t b = get();
  cudaEventRecord(b, s);
  std::lock_guard<std::mutex> g(mu);
  pending.push_back({a, b, klass, fl, by, nl});
}
void Profiler::collect() {
  std::lock_guard<std::mutex> g(mu);
  for (auto& r : pending) {
    float t = 0.f;
    cudaEventSynchronize(r.b);
    cudaEventElapsedTime(&t, r.a, r.b);
    ms[r.klass] += t;
    flops[r.klass] += r.flops;
    bytes[r.klass] += r.bytes;
    launches[r.klass] += r.launches;
    pool.push_back(r.a);
    pool.push_back(r.b);
  }
  pending.clear();
}
void Profiler::reset() {
  collect();
  for (int i = 0; i < KC_N; ++i) ms[i] = flops[i] = bytes[i] = 0, launches[i] = 0;
}
Profiler::~Profiler() {
  for (auto& r : pending) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : pool) cudaEventDestroy(e);
}

namespace {

struct Scoped {
  Profiler& p;
  cudaStream_t s;
  int klass;
  double fl, by;
  cudaEvent_t a = nullptr;
  int n = 0;
  bool count = true;  // false: a nested sub-class record (the launches are counted by the outer one)
  Scoped(Profiler& p_, cudaStream_t s_, int k, double f, double b) : p(p_), s(s_), klass(k), fl(f), by(b) {
    if (klass >= 0) p.begin(s, &a);
  }
  void launched(int c) {
    if (c < 0) fail(FRAG_E_CONTRACT, "kernel launch rejected the shape");
    n += c;
    if (count) g_launches += (uint64_t)c;
  }
  ~Scoped() {
    if (p.on && klass >= 0) p.end(s, a, klass, fl, by, n);
  }
};

// split-K / stream-K tile counters: the last 2 * CHAIN_MAX_OPS ints of
// gemm_cnt are the GEMM chain's done / exit counters and never handed out
inline int gemm_counter_cap(const Result* r) {
  return (int)(r->gemm_cnt.bytes / sizeof(int)) - 2 * fragk::CHAIN_MAX_OPS;
}

inline void peek(const char* what) {
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(FRAG_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

}  // namespace

uint64_t weight_seed(uint64_t seed, int tensor_id) {
  return mix64(seed + 0x9e3779b97f4a7c15ULL * (uint64_t)(tensor_id + 1));
}

// ---------------------------------------------------------------- engine
void Engine::ensure_rope(int rows) {
  std::lock_guard<std::mutex> g(rope_mu);
  if (rows <= rope_rows) return;
  const int half = cfg.head_dim / 2;
  int n = rows < 4096 ? 4096 : rows;
  std::vector<float2> tab((size_t)n * half);
  for (int r = 0; r < n; ++r) {
    const double pos = (double)(r + 1);
    for (int i = 0; i < half; ++i) {
      const double a = pos * theta[i];
      tab[(size_t)r * half + i] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
  }
  DeviceGuard dg(device);
  cudaDeviceSynchronize();  // the table may be in use by in-flight work
  rope.alloc(tab.size() * sizeof(float2));
  check_cuda(cudaMemcpy(rope.p, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice), "rope upload");
  rope_rows = n;
}

static void validate_cfg(const frag_model_cfg& c) {
  auto req = [](bool ok, const char* m) {
    if (!ok) fail(FRAG_E_CONTRACT, std::string("invalid ModelConfig: ") + m);
  };
  req(c.layers >= 1, "layers >= 1");
  req(c.head_dim == 64 || c.head_dim == 128, "head_dim in {64, 128}");
  req(c.n_heads >= 1 && c.n_kv_heads >= 1 && c.n_heads % c.n_kv_heads == 0, "n_heads multiple of n_kv_heads");
  req(128 % (c.n_heads / c.n_kv_heads) == 0, "GQA group divides 128");
  req(c.d_model % 64 == 0, "d_model % 64 == 0");
  req(c.ffn_dim % 64 == 0, "ffn_dim % 64 == 0");
  req(c.vocab % 64 == 0 && c.vocab >= 2, "vocab % 64 == 0");
  req((c.n_heads * c.head_dim) % 64 == 0, "n_heads*head_dim % 64 == 0");
  req(c.rope_base > 0, "rope_base > 0");
  req(c.norm_eps > 0, "norm_eps > 0");
}

Engine* engine_create(const frag_model_cfg& cfg, int device, uint64_t seed) {
  validate_cfg(cfg);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    fail(FRAG_E_CUDA, "no CUDA device available (this library has no CPU fallback)");
  }
  if (device < 0 || device >= ndev) fail(FRAG_E_CONTRACT, "device ordinal out of range");
  DeviceGuard dg(device);
  auto e = std::make_unique<Engine>();
  e->cfg = cfg;
  e->device = device;
  e->seed = seed;
  const size_t d = cfg.d_model, V = cfg.vocab, F = cfg.ffn_dim, qc = (size_t)cfg.n_heads * cfg.head_dim;
  const size_t qkv = e->qkv_cols();
  // carve one allocation
  std::vector<size_t> sizes = {V * d, V * d, d};
  for (int l = 0; l < cfg.layers; ++l) {
    sizes.push_back(qkv * d);
    sizes.push_back(d * qc);
    sizes.push_back(2 * F * d);
    sizes.push_back(d * F);
    sizes.push_back(d);
    sizes.push_back(d);
  }
  size_t total = 0;
  std::vector<size_t> offs;
  for (size_t s : sizes) {
    offs.push_back(total);
    total += align_up(s * sizeof(bf16), 256);
    e->n_params += s;
  }
  e->weights.alloc(total);
  bf16* base = e->weights.as<bf16>();
  auto at = [&](size_t i) { return reinterpret_cast<bf16*>(reinterpret_cast<char*>(base) + offs[i]); };
  e->emb = at(0);
  e->lm_head = at(1);
  e->final_norm = at(2);
  e->layers.resize(cfg.layers);
  for (int l = 0; l < cfg.layers; ++l) {
    auto& L = e->layers[l];
    L.wqkv = at(3 + 6 * l);
    L.wo = at(4 + 6 * l);
    L.wgu = at(5 + 6 * l);
    L.wd = at(6 + 6 * l);
    L.attn_norm = at(7 + 6 * l);
    L.ffn_norm = at(8 + 6 * l);
  }
  cudaStream_t s;
  check_cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  const float sig = 0.02f;
  // init_model: tensor ids 0 emb, 1 lm_head, 16+8l+{0..6} wq wk wv wo wg wu wd
  fragk::init_normal_bf16(e->emb, weight_seed(seed, 0), V, d, sig, (int)V, 0, 0, s);
  fragk::init_normal_bf16(e->lm_head, weight_seed(seed, 1), V, d, sig, (int)V, 0, 0, s);
  fragk::fill_bf16(e->final_norm, d, 1.0f, s);
  const int Hq = cfg.n_heads, Hkv = cfg.n_kv_heads, dh = cfg.head_dim;
  for (int l = 0; l < cfg.layers; ++l) {
    auto& L = e->layers[l];
    const int t0 = 16 + 8 * l;
    const int qrows = Hq * dh, krows = Hkv * dh;
    fragk::init_normal_bf16(L.wqkv, weight_seed(seed, t0 + 0), qrows, d, sig, qrows, 0, 0, s);
    fragk::init_normal_bf16(L.wqkv, weight_seed(seed, t0 + 1), krows, d, sig, krows, 0, qrows, s);
    fragk::init_normal_bf16(L.wqkv, weight_seed(seed, t0 + 2), krows, d, sig, krows, 0, qrows + krows, s);
    fragk::init_normal_bf16(L.wo, weight_seed(seed, t0 + 3), d, qc, sig, (int)d, 0, 0, s);
    // gate/up interleaved in 32-row blocks: packed row = (r/32)*64 + {0 | 32} + r%32
    fragk::init_normal_bf16(L.wgu, weight_seed(seed, t0 + 4), F, d, sig, 32, 64, 0, s);
    fragk::init_normal_bf16(L.wgu, weight_seed(seed, t0 + 5), F, d, sig, 32, 64, 32, s);
    fragk::init_normal_bf16(L.wd, weight_seed(seed, t0 + 6), d, F, sig, (int)d, 0, 0, s);
    fragk::fill_bf16(L.attn_norm, d, 1.0f, s);
    fragk::fill_bf16(L.ffn_norm, d, 1.0f, s);
  }
  g_launches += 3 + 9 * (uint64_t)cfg.layers;
  check_cuda(cudaStreamSynchronize(s), "weight init");
  cudaStreamDestroy(s);
  const int half = dh / 2;
  e->theta.resize(half);
  for (int i = 0; i < half; ++i) e->theta[i] = std::pow(cfg.rope_base, -2.0 * (double)(i + 1) / (double)dh);
  e->ensure_rope(4096);
  return e.release();
}

Result::~Result() {
  for (auto& g : graphs)
    if (g.second.exec) cudaGraphExecDestroy(g.second.exec);
  if (cap_stream) cudaStreamDestroy(cap_stream);
  if (side) cudaStreamDestroy(side);
  if (fork_ev) cudaEventDestroy(fork_ev);
  for (auto& e : layer_ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : vwin_ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : ev)
    if (e) cudaEventDestroy(e);
}

void result_init(Result* r, Engine* e, int max_tokens) {
  if (max_tokens < 1) fail(FRAG_E_CONTRACT, "max_tokens must be positive");
  DeviceGuard dg(e->device);
  const auto& c = e->cfg;
  r->eng = e;
  r->max_tokens = max_tokens;
  const size_t kvc = (size_t)c.n_kv_heads * c.head_dim, qc = (size_t)c.n_heads * c.head_dim;
  const size_t M = max_tokens;
  r->k_fused.alloc((size_t)c.layers * M * kvc * sizeof(bf16));  // V: use_private_v / shared pages
  r->h.alloc(M * c.d_model * sizeof(float));
  r->x.alloc(M * std::max<size_t>(c.d_model, qc) * sizeof(bf16));
  r->q.alloc(M * qc * sizeof(bf16));
  r->attn.alloc(M * qc * sizeof(bf16));
  r->act.alloc(M * c.ffn_dim * sizeof(bf16));
  r->plan_rows.alloc(M * sizeof(int));
  r->plan_tok.alloc(M * sizeof(int));
  r->chunk_tok.alloc(M * sizeof(int));
  r->q_tok.alloc(M * sizeof(int));
  r->scores.alloc(M * sizeof(float));
  r->row_map.alloc(M * sizeof(int));
  r->ssq.alloc((size_t)(c.d_model / 32) * M * sizeof(float));  // folded RMSNorm partials
  // split-K workspace (small-M GEMMs) + self-resetting tile counters
  r->gemm_ws.alloc((size_t)32 << 20);
  r->gemm_cnt.alloc(16384 * sizeof(int));
  check_cuda(cudaMemset(r->gemm_cnt.p, 0, r->gemm_cnt.bytes), "counter init");
  for (auto& ev : r->ev) check_cuda(cudaEventCreate(&ev), "cudaEventCreate");
  e->ensure_rope(max_tokens);
}

// FRAG_SHARED_V=0 keeps every request's V private (the r01 layout).
std::atomic<int> g_shared_v{-1};  // -1: not read from the environment yet
bool shared_v_enabled() {
  int v = g_shared_v.load(std::memory_order_relaxed);
  if (v < 0) {
    const char* ev = std::getenv("FRAG_SHARED_V");
    int want = (ev && ev[0] == '0') ? 0 : 1;
    g_shared_v.compare_exchange_strong(v, want);
    v = g_shared_v.load(std::memory_order_relaxed);
  }
  return v != 0;
}

int set_shared_v(int on) {
  const int prev = shared_v_enabled() ? 1 : 0;
  if (on >= 0) g_shared_v.store(on ? 1 : 0);
  return prev;
}

uint64_t result_device_bytes(const Result* r) {
  uint64_t b = 0;
  for (const DevBuf* d : {&r->k_fused, &r->v_fused, &r->h, &r->x, &r->q, &r->attn, &r->act, &r->plan_rows,
                          &r->plan_tok, &r->chunk_tok, &r->q_tok, &r->q_final, &r->scores, &r->part_ms, &r->row_ms,
                          &r->part_o, &r->part_lse, &r->logits, &r->row_map, &r->stitch_desc, &r->stitch_tab,
                          &r->lm_x, &r->gemm_ws, &r->gemm_cnt, &r->dec_tok, &r->fr_save, &r->dev, &r->score_col,
                          &r->score_q, &r->ssq, &r->vx, &r->vx_map, &r->vseg, &r->vplan_args, &r->vplan_tile, &r->vplan_prim,
                          &r->vplan_ent, &r->vwin})
    b += d->bytes;
  return b;
}

void use_private_v(Result* r) {
  const auto& c = r->eng->cfg;
  r->vshared = false;
  r->v_materialized = false;
  r->vrefs.clear();
  r->vseq.clear();
  r->v_tail_row0 = 0x7fffffff;
  r->v_tail_slot0 = 0;
  r->v_fused.ensure((size_t)c.layers * r->max_tokens * c.n_kv_heads * c.head_dim * sizeof(bf16));
}

void materialize_v(Result* r, cudaStream_t s) {
  if (!r->vshared || r->v_materialized) return;
  const auto& c = r->eng->cfg;
  const size_t kvc = (size_t)c.n_kv_heads * c.head_dim;
  r->v_fused.ensure((size_t)c.layers * r->max_tokens * kvc * sizeof(bf16));
  for (const auto& q : r->vseq) {
    const int rows = q.T;  // cache rows of the sequence (incl. decoded tokens)
    const int rc = fragk::vpage_gather(r->vseg.as<fragk::VSeg>() + q.seg0, r->vplan_tile.as<int>() + q.vt_off,
                                       r->vplan_prim.as<int2>() + q.vp_off,
                                       r->vplan_ent.as<unsigned long long>() + q.ve_off, r->vx.as<bf16>(),
                                       (size_t)r->vx_rows * kvc, q.tail_row0, q.tail_slot_s, rows, c.layers, (int)kvc,
                                       r->v_fused.as<bf16>() + (size_t)q.base * kvc, (size_t)r->max_tokens * kvc, s);
    if (rc < 0) fail(FRAG_E_CUDA, "shared V read-back launch failed");
  }
  check_cuda(cudaStreamSynchronize(s), "shared V read-back");
  r->v_materialized = true;
}

// ---------------------------------------------------------------- run_rows
void run_rows(Engine* e, Result* r, cudaStream_t s, int M, int T, PassMode mode, const int* row_map_dev,
              int n_logit_rows, int n_layers, const cudaEvent_t* layer_ready, const std::vector<Seg>* segs_in,
              int keep_last) {
  if (M <= 0) return;
  const auto& c = e->cfg;
  const int L = (n_layers > 0 && n_layers < c.layers) ? n_layers : c.layers;
  const int d = c.d_model, Hq = c.n_heads, Hkv = c.n_kv_heads, dh = c.head_dim, F = c.ffn_dim;
  const size_t qc = (size_t)Hq * dh, kvc = (size_t)Hkv * dh, qkv = e->qkv_cols();
  const size_t lstride = (size_t)r->max_tokens * kvc;
  Profiler& P = e->prof;
  bf16* kf = r->k_fused.as<bf16>();
  bf16* vf = r->vshared ? nullptr : r->v_fused.as<bf16>();
  const int* prow = r->plan_rows.as<int>();
  const int* ptok = r->plan_tok.as<int>();
  float* h = r->h.as<float>();
  bf16* x = r->x.as<bf16>();
  // RMSNorm folded into the GEMM epilogues (EpiParams::ssq_*; FRAG_FUSED_NORM=0
  // runs the standalone rmsnorm kernel instead). Layer 0's norm stays in the
  // embedding kernel; the final norm stays standalone (row gather for lm_head).
  // The norm gains are 1 (init_model) -- a non-unit gain would
  // be folded into the weights' input columns at engine creation.
  static const bool fuse_norm = [] {
    const char* v = std::getenv("FRAG_FUSED_NORM");
    return !(v && v[0] == '0');
  }();
  float* ssq = r->ssq.as<float>();
  const int ssq_ld = r->max_tokens;
  auto norm_in = [&](fragk::EpiParams& ep, size_t row0) {
    ep.ssq_in = ssq + row0;
    ep.ssq_ld = ssq_ld;
    ep.ssq_n = d / 32;
    ep.norm_d = d;
    ep.norm_eps = c.norm_eps;
  };
  auto norm_out = [&](fragk::EpiParams& ep, size_t row0) {
    ep.ssq_out = ssq + row0;
    ep.ssq_ld = ssq_ld;
    ep.x_out = x + row0 * d;
  };
  auto with_ws = [&](fragk::EpiParams& ep) {
    ep.ws = r->gemm_ws.as<float>();
    ep.ws_bytes = r->gemm_ws.bytes;
    ep.counters = r->gemm_cnt.as<int>();
    ep.counters_cap = gemm_counter_cap(r);
  };

  // one sequence unless batched (segments of plan rows, each over its own
  // slice of the fused cache starting at cache row `base`)
  const std::vector<Seg> one{Seg{0, M, 0, T}};
  const std::vector<Seg>& segs = segs_in ? *segs_in : one;
  // split-KV policy per segment, splits of >= 256 keys: very few query blocks
  // (question pass, decode) fill exactly one wave (the attention CTA takes a
  // whole SM); otherwise >= 2 waves
  const int G = Hq / Hkv;
  const int tpc = fragk::attn_rows_per_cta() / G;  // tokens per attention CTA
  const int sms = fragk::num_sms();
  auto split_policy = [&](int Ms, int Ts, int& n_splits, int& split_keys) {
    const int nqb = (Ms + tpc - 1) / tpc;
    const long ctas = (long)nqb * Hkv;
    n_splits = 1, split_keys = 0;
    if (ctas < 2L * sms && Ts > 512) {
      n_splits = ctas <= sms / 2 ? (int)(sms / ctas) : (int)((2L * sms + ctas - 1) / ctas);
      const int max_splits = (Ts + 255) / 256;
      if (n_splits > max_splits) n_splits = max_splits;
      if (n_splits > 64) n_splits = 64;  // the combine kernel's limit
      split_keys = (int)align_up((size_t)((Ts + n_splits - 1) / n_splits), 128);
      n_splits = (Ts + split_keys - 1) / split_keys;
      if (n_splits <= 1) n_splits = 1, split_keys = 0;
    }
  };
  std::vector<std::pair<int, int>> seg_split(segs.size());
  for (size_t i = 0; i < segs.size(); ++i) {
    split_policy(segs[i].M, segs[i].T, seg_split[i].first, seg_split[i].second);
    if (seg_split[i].first > 1) {
      r->part_o.ensure((size_t)seg_split[i].first * segs[i].M * qc * sizeof(float));
      r->part_lse.ensure((size_t)seg_split[i].first * segs[i].M * Hq * sizeof(float));
    }
  }
  // shared V pages: a large pass (more query rows than one attention tile: the
  // sparse pass, long or batched questions) stages each layer's V into a
  // double-buffered window at its cache rows -- records copied by vwindow_fill
  // before that layer's QKV, fresh rows added by the QKV epilogue -- and reads
  // it like a private cache; small passes (the question pass of <= 128/G
  // tokens, r = 0, decode) patch the record tiles inside the attention kernel
  const bool vwin = r->vshared && M > 128 / (Hq / Hkv);
  const size_t wstride = (size_t)r->max_tokens * kvc;
  // The fills run on the side stream, two layers ahead: layer l+2's fill waits
  // only for layer l's attention (the last reader of its buffer) and overlaps
  // the tensor-bound GEMMs; a layer's QKV waits for its window.
  static const bool vwin_side = [] {  // FRAG_VWIN_SIDE=0: fills in the request stream before each QKV
    const char* v = std::getenv("FRAG_VWIN_SIDE");
    return !(v && v[0] == '0');
  }();
  if (vwin) {
    r->vwin.ensure(2 * wstride * sizeof(bf16));  // first (eager) request of a shape allocates
    if (!r->side) check_cuda(cudaStreamCreateWithFlags(&r->side, cudaStreamNonBlocking), "side stream");
    while ((int)r->vwin_ev.size() < 2 * L) {
      cudaEvent_t ev;
      check_cuda(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "window event");
      r->vwin_ev.push_back(ev);
    }
  }
  auto vwin_fill = [&](int l, cudaStream_t fs) {
    Scoped sc(P, fs, KC_VWIN, 0, 4.0 * (double)r->vseg_rows * kvc);  // read + write, bf16
    const int rc = fragk::vwindow_fill(r->vseg.as<fragk::VSeg>(), r->vseg_n, r->vseg_max_rows, l, (int)kvc,
                                       r->vwin.as<bf16>() + (size_t)(l & 1) * wstride, fs);
    if (rc < 0) fail(FRAG_E_CUDA, "V window launch failed");
    sc.launched(rc);
  };
  auto vwin_side_fill = [&](int l) {  // on the side stream, after layer l-2's attention (or the pass start)
    if (!vwin || !vwin_side || l >= L) return;
    cudaEvent_t after = l >= 2 ? r->vwin_ev[l - 2] : r->vwin_ev[L + l];  // [L + l]: pass-start fork
    if (l < 2) check_cuda(cudaEventRecord(after, s), "window fork");
    check_cuda(cudaStreamWaitEvent(r->side, after, 0), "window wait");
    vwin_fill(l, r->side);
    check_cuda(cudaEventRecord(r->vwin_ev[L + l], r->side), "window filled");
  };
  auto vwin_join = [&](int l) {  // before layer l's QKV
    if (!vwin) return;
    if (vwin_side)
      check_cuda(cudaStreamWaitEvent(s, r->vwin_ev[L + l], 0), "window join");
    else
      vwin_fill(l, s);
  };
  auto vwin_attn_done = [&](int l) {  // after layer l's attention: its buffer goes to layer l + 2
    if (!vwin || !vwin_side) return;
    check_cuda(cudaEventRecord(r->vwin_ev[l], s), "window free");
    vwin_side_fill(l + 2);
  };
  vwin_side_fill(0);
  vwin_side_fill(1);
  const bool want_qf = mode == PASS_QUESTION || (mode == PASS_FULL && r->q_final_in_full);
  if (want_qf) r->q_final.ensure((size_t)M * qc * sizeof(float));

  {
    Scoped sc(P, s, KC_NORM, 0, (double)M * d * (2 + 4 + 2));
    fragk::embed_rmsnorm(e->emb, ptok, M, d, e->layers[0].attn_norm, c.norm_eps, h, x, s);
    sc.launched(1);
  }
  auto qkv_ep = [&](int l) {
    fragk::EpiParams ep;
    with_ws(ep);
    ep.rows = prow;
    ep.rope = e->rope.as<float2>();
    ep.q_out = r->q.as<bf16>();
    ep.q_out_f32 = (want_qf && l == L - 1) ? r->q_final.as<float>() : nullptr;
    ep.k_cache = kf + l * lstride;
    if (r->vshared) {  // fresh V -> exclusive slots (and the staged window)
      ep.v_cache = r->vx.as<bf16>() + (size_t)l * r->vx_rows * kvc;
      ep.v_slots = 1;
      ep.v_tail_row0 = r->v_tail_row0;
      ep.v_tail_slot0 = r->v_tail_slot0;
      if (vwin) ep.v_cache2 = r->vwin.as<bf16>() + (size_t)(l & 1) * wstride;
    } else {
      ep.v_cache = vf + l * lstride;
    }
    ep.rows_per_seq = r->rows_per_seq;
    ep.Hq = Hq;
    ep.Hkv = Hkv;
    ep.dh = dh;
    if (l > 0 && fuse_norm) norm_in(ep, 0);
    return ep;
  };
  // <= 128 rows (question pass, decode, r = 0): the O -> gate/up -> down ->
  // next-QKV projections of a layer run as one persistent GEMM chain
  // (gemm_chain.cu; FRAG_GEMM_CHAIN=0 launches them one by one)
  static const bool chain_env = [] {
    const char* v = std::getenv("FRAG_GEMM_CHAIN");
    return !(v && v[0] == '0');
  }();
  const bool use_chain = chain_env && fuse_norm && fragk::gemm_chain_supported(M, (int)qkv, d) &&
                         fragk::gemm_chain_supported(M, d, (int)qc) && fragk::gemm_chain_supported(M, 2 * F, d) &&
                         fragk::gemm_chain_supported(M, d, F);
  int* chain_done = r->gemm_cnt.as<int>() + (r->gemm_cnt.bytes / sizeof(int) - 2 * fragk::CHAIN_MAX_OPS);
  // shared V pages: the attention of sequence g.seq reads V through its plan
  auto vattn = [&](fragk::AttnArgs& a, const Seg& g, int l) {
    if (vwin) {
      a.v = r->vwin.as<bf16>() + (size_t)(l & 1) * wstride + (size_t)g.base * kvc;
      return;
    }
    if (!r->vshared) return;
    const Result::VSeq& q = r->vseq[g.seq];
    a.v = nullptr;
    a.vsegs = r->vseg.as<fragk::VSeg>() + q.seg0;
    a.n_vseg = q.n_seg;
    a.vtile = r->vplan_tile.as<int>() + q.vt_off;
    a.vprim = r->vplan_prim.as<int2>() + q.vp_off;
    a.vent = r->vplan_ent.as<unsigned long long>() + q.ve_off;
    a.vx = r->vx.as<bf16>() + (size_t)l * r->vx_rows * kvc;
    a.vx_map = r->vx_map.as<CUtensorMap>();
    a.layer = l;
    a.tail_row0 = q.tail_row0;
    a.tail_slot0 = mode == PASS_QUESTION ? q.tail_slot_q : q.tail_slot_s;
  };
  bool qkv_done = false;  // this layer's QKV already ran inside the previous layer's chain
  for (int l = 0; l < L; ++l) {
    const auto& W = e->layers[l];
    if (l > 0 && !fuse_norm) {
      Scoped sc(P, s, KC_NORM, 0, (double)M * d * (4 + 2));
      fragk::rmsnorm(h, M, d, W.attn_norm, c.norm_eps, x, s);
      sc.launched(1);
    }
    if (!qkv_done) {
      vwin_join(l);
      fragk::EpiParams ep = qkv_ep(l);
      Scoped sc(P, s, gemm_class(M), 2.0 * M * qkv * d, 2.0 * (qkv * d + (double)M * (d + qkv)));
      sc.launched(fragk::gemm_bf16_tc(x, W.wqkv, M, (int)qkv, d, fragk::EPI_QKV, ep, s));
    }
    qkv_done = false;
    if (mode != PASS_FULL && l == L - 1) break;
    if (layer_ready) check_cuda(cudaStreamWaitEvent(s, layer_ready[l], 0), "wait stitched layer");
    // Last layer: every row's K/V are in the cache now (the QKV epilogue), and
    // only the trailing keep_last rows' hidden states feed anything (the
    // logits); the other rows' last-layer attention, O projection and MLP have
    // no consumer, so the rest of the layer runs on those rows only.
    const bool prune = mode == PASS_FULL && l == c.layers - 1 && keep_last > 0 && keep_last < M && !segs_in;
    // batched: keep the last row of every sequence, compacted into the rows
    // [M, M + n_seq) of the workspaces (their order = the sequences')
    const bool seg_prune = mode == PASS_FULL && l == c.layers - 1 && keep_last < 0 && segs_in &&
                           M + (int)segs.size() <= r->max_tokens;
    const int Ml = prune ? keep_last : (seg_prune ? (int)segs.size() : M);
    const size_t off = prune ? (size_t)(M - Ml) : (seg_prune ? (size_t)M : 0);
    if (seg_prune) {
      for (size_t si = 0; si < segs.size(); ++si) {
        const Seg& g = segs[si];
        const size_t src = (size_t)g.off + g.M - 1;
        check_cuda(cudaMemcpyAsync(h + (off + si) * d, h + src * d, d * sizeof(float), cudaMemcpyDeviceToDevice, s),
                   "gather last rows");
        int ns, sk;
        split_policy(1, g.T, ns, sk);
        if (ns > 1) {
          r->part_o.ensure((size_t)ns * qc * sizeof(float));
          r->part_lse.ensure((size_t)ns * Hq * sizeof(float));
        }
        fragk::AttnArgs a{};
        a.q = r->q.as<bf16>() + src * qc;
        a.k = kf + l * lstride + (size_t)g.base * kvc;
        a.v = vf + l * lstride + (size_t)g.base * kvc;
        a.rows = prow + src;
        a.row_base = g.base;
        a.out = r->attn.as<bf16>() + (off + si) * qc;
        a.part_o = r->part_o.as<float>();
        a.part_lse = r->part_lse.as<float>();
        a.M = 1;
        a.T = g.T;
        a.Hq = Hq;
        a.Hkv = Hkv;
        a.dh = dh;
        a.split_keys = sk;
        a.n_splits = ns;
        a.scale = 1.0f / std::sqrt((float)dh);
        vattn(a, g, l);
        Scoped sc(P, s, KC_ATTN, 0, 0);
        sc.launched(fragk::sparse_q_attention(a, s));
      }
    }
    std::vector<Seg> last_seg;
    std::vector<std::pair<int, int>> last_split;
    if (prune) {
      last_seg.push_back(Seg{(int)off, Ml, 0, T, 0});
      last_split.resize(1);
      split_policy(Ml, T, last_split[0].first, last_split[0].second);
      if (last_split[0].first > 1) {
        r->part_o.ensure((size_t)last_split[0].first * Ml * qc * sizeof(float));
        r->part_lse.ensure((size_t)last_split[0].first * Ml * Hq * sizeof(float));
      }
    }
    static const std::vector<Seg> no_segs;
    const std::vector<Seg>& asegs = prune ? last_seg : (seg_prune ? no_segs : segs);
    const std::vector<std::pair<int, int>>& asplit = prune ? last_split : seg_split;
    // the layer's projections run as a GEMM chain: a single sequence's
    // split-KV combine moves into the chain (pre-op writing op 0's A rows)
    const bool chain_layer = use_chain && Ml == M && off == 0;
    const bool defer_ok = chain_layer && asegs.size() == 1;
    bool deferred = false;
    fragk::AttnArgs deferred_args{};
    for (size_t si = 0; si < asegs.size(); ++si) {
      const Seg& g = asegs[si];
      if (g.M <= 0) continue;
      fragk::AttnArgs a{};
      a.q = r->q.as<bf16>() + (size_t)g.off * qc;
      a.k = kf + l * lstride + (size_t)g.base * kvc;
      a.v = vf + l * lstride + (size_t)g.base * kvc;
      a.rows = prow + g.off;
      a.row_base = g.base;
      a.out = r->attn.as<bf16>() + (size_t)g.off * qc;
      a.part_o = r->part_o.as<float>();
      a.part_lse = r->part_lse.as<float>();
      a.M = g.M;
      a.T = g.T;
      a.Hq = Hq;
      a.Hkv = Hkv;
      a.dh = dh;
      a.split_keys = asplit[si].second;
      a.n_splits = asplit[si].first;
      a.scale = 1.0f / std::sqrt((float)dh);
      vattn(a, g, l);
      Scoped sc(P, s, KC_ATTN, 0, 0);
      sc.launched(fragk::sparse_q_attention(a, s, defer_ok ? &deferred : nullptr));
      if (deferred) deferred_args = a;
    }
    vwin_attn_done(l);
    if (chain_layer) {
      fragk::ChainStep st[fragk::CHAIN_MAX_OPS];
      int n = 0;
      st[n].A = r->attn.as<bf16>(), st[n].B = W.wo, st[n].N = d, st[n].K = (int)qc, st[n].epi = fragk::EPI_RESID;
      with_ws(st[n].ep);
      st[n].ep.resid = h, st[n].ep.ldo = d;
      norm_out(st[n].ep, 0);
      ++n;
      st[n].A = x, st[n].B = W.wgu, st[n].N = 2 * F, st[n].K = d, st[n].epi = fragk::EPI_SWIGLU;
      with_ws(st[n].ep);
      st[n].ep.out_bf16 = r->act.as<bf16>(), st[n].ep.ldo = F;
      norm_in(st[n].ep, 0);
      ++n;
      st[n].A = r->act.as<bf16>(), st[n].B = W.wd, st[n].N = d, st[n].K = F, st[n].epi = fragk::EPI_RESID;
      with_ws(st[n].ep);
      st[n].ep.resid = h, st[n].ep.ldo = d;
      if (l + 1 < L) norm_out(st[n].ep, 0);
      ++n;
      double flop = 2.0 * M * d * qc + 2.0 * M * 2.0 * F * d + 2.0 * M * (double)d * F;
      double bytes = 2.0 * (qc * d + 2.0 * F * d + (double)F * d);
      if (l + 1 < L) {
        vwin_join(l + 1);
        st[n].A = x, st[n].B = e->layers[l + 1].wqkv, st[n].N = (int)qkv, st[n].K = d;
        st[n].epi = fragk::EPI_QKV;
        st[n].ep = qkv_ep(l + 1);
        ++n;
        flop += 2.0 * M * qkv * d;
        bytes += 2.0 * qkv * d;
        qkv_done = true;
      }
      Scoped sc(P, s, gemm_class(M), flop, bytes);
      sc.launched(fragk::gemm_chain_tc(st, n, M, chain_done, s, deferred ? &deferred_args : nullptr));
      peek("layer");
      continue;
    }
    {
      fragk::EpiParams ep;
      with_ws(ep);
      ep.resid = h + off * d;
      ep.ldo = d;
      if (fuse_norm) norm_out(ep, off);
      Scoped sc(P, s, gemm_class(Ml), 2.0 * Ml * d * qc, 2.0 * (qc * d + (double)Ml * qc) + 8.0 * Ml * d);
      sc.launched(fragk::gemm_bf16_tc(r->attn.as<bf16>() + off * qc, W.wo, Ml, d, (int)qc, fragk::EPI_RESID, ep, s));
    }
    if (!fuse_norm) {
      Scoped sc(P, s, KC_NORM, 0, (double)Ml * d * (4 + 2));
      fragk::rmsnorm(h + off * d, Ml, d, W.ffn_norm, c.norm_eps, x + off * d, s);
      sc.launched(1);
    }
    {
      fragk::EpiParams ep;
      with_ws(ep);
      ep.out_bf16 = r->act.as<bf16>() + off * F;
      ep.ldo = F;
      if (fuse_norm) norm_in(ep, off);
      const double gu_flop = 2.0 * Ml * 2.0 * F * d, gu_bytes = 2.0 * (2.0 * F * d + (double)Ml * d + (double)Ml * F);
      Scoped sc(P, s, gemm_class(Ml), gu_flop, gu_bytes);
      // the single largest GEMM of the sparse pass also gets its own class (the
      // bench's roofline kernel): nested events, a subset of KC_GEMM
      Scoped sc_gu(P, s, gemm_class(Ml) == KC_GEMM ? KC_GEMM_GU : -1, gu_flop, gu_bytes);
      sc_gu.count = false;
      const int nl = fragk::gemm_bf16_tc(x + off * d, W.wgu, Ml, 2 * F, d, fragk::EPI_SWIGLU, ep, s);
      sc_gu.launched(nl);
      sc.launched(nl);
    }
    {
      fragk::EpiParams ep;
      with_ws(ep);
      ep.resid = h + off * d;
      ep.ldo = d;
      if (fuse_norm && l + 1 < L) norm_out(ep, off);  // feeds the next layer's QKV
      Scoped sc(P, s, gemm_class(Ml), 2.0 * Ml * (double)d * F,
                2.0 * ((double)F * d + (double)Ml * F) + 8.0 * Ml * d);
      sc.launched(fragk::gemm_bf16_tc(r->act.as<bf16>() + off * F, W.wd, Ml, d, F, fragk::EPI_RESID, ep, s));
    }
    peek("layer");
  }
  if (mode == PASS_FULL && n_logit_rows > 0 && L == c.layers) {
    r->lm_x.ensure((size_t)n_logit_rows * d * sizeof(bf16));
    r->logits.ensure((size_t)n_logit_rows * c.vocab * sizeof(float));
    {
      Scoped sc(P, s, KC_NORM, 0, (double)n_logit_rows * d * 6);
      fragk::rmsnorm(h, n_logit_rows, d, e->final_norm, c.norm_eps, r->lm_x.as<bf16>(), s, row_map_dev);
      sc.launched(1);
    }
    fragk::EpiParams ep;
    with_ws(ep);
    ep.out_f32 = r->logits.as<float>();
    ep.ldo = c.vocab;
    Scoped sc(P, s, gemm_class(n_logit_rows), 2.0 * n_logit_rows * (double)c.vocab * d, 2.0 * c.vocab * (double)d);
    sc.launched(fragk::gemm_bf16_tc(r->lm_x.as<bf16>(), e->lm_head, n_logit_rows, c.vocab, d,
                                    fragk::EPI_STORE_F32, ep, s));
  }
  peek("run_rows");
}

// ---------------------------------------------------------------- helpers
namespace {

struct PinGuard {
  Store* st;
  std::vector<frag_chunk_id> ids;
  ~PinGuard() {
    for (auto& id : ids) {
      try {
        store_release(st, id);
      } catch (...) {
      }
    }
  }
};

// Bump allocator over the result's pinned staging buffer.
struct Stage {
  PinnedBuf& buf;
  size_t off = 0;
  explicit Stage(PinnedBuf& b) : buf(b) {}
  template <class T>
  T* take(size_t n) {
    off = align_up(off, 64);
    T* p = reinterpret_cast<T*>(static_cast<char*>(buf.p) + off);
    off += n * sizeof(T);
    if (off > buf.bytes) fail(FRAG_E_CONTRACT, "staging overflow");
    return p;
  }
};

// K1 host side: per-chunk descriptors and cos/sin(delta*theta) tables staged and
// copied to the device (per request); the kernel launch is part of the body.
// One part per sequence: its KV_S and records placed from cache row `base`
// (base > 0 only for batched requests sharing one fused cache).
struct StitchPart {
  const SysKV* sys;
  const std::vector<Record*>* recs;
  int S, base;
};
StitchPlan stitch_prepare_parts(Engine* e, Result* r, cudaStream_t s, Stage& stg, const std::vector<StitchPart>& parts) {
  const auto& c = e->cfg;
  const int half = c.head_dim / 2;
  StitchPlan p;
  for (const auto& pt : parts) p.n_desc += (pt.sys && pt.sys->n > 0 ? 1 : 0) + (int)pt.recs->size();
  if (p.n_desc == 0) return p;
  auto* desc = stg.take<fragk::StitchChunk>(p.n_desc);
  std::vector<float2> tabs;
  int nd = 0, n_tab = 0;
  const size_t kvc = (size_t)c.n_kv_heads * c.head_dim;
  for (const auto& pt : parts) {
    if (pt.sys && pt.sys->n > 0) {
      desc[nd++] = {pt.sys->kv.as<bf16>(), pt.sys->kv.as<bf16>() + (size_t)c.layers * pt.sys->n * kvc, pt.sys->n,
                    pt.base, -1};
      if (pt.sys->n > p.max_rows) p.max_rows = pt.sys->n;
    }
    int row = pt.S;  // local row = position - 1
    for (Record* rec : *pt.recs) {
      const int target_start = row + 1;  // 1-based
      const int delta = target_start - rec->native_start;
      int table = -1;
      if (delta != 0) {
        // shift_rope = apply_rope(v, new - old): cos/sin(delta * theta_i), fp64 angles
        table = n_tab++;
        for (int i = 0; i < half; ++i) {
          const double ang = (double)delta * e->theta[i];
          tabs.push_back(make_float2((float)std::cos(ang), (float)std::sin(ang)));
        }
      }
      desc[nd++] = {rec->k(), rec->v(), rec->n_tok, pt.base + row, table};
      if (rec->n_tok > p.max_rows) p.max_rows = rec->n_tok;
      row += rec->n_tok;
    }
  }
  float2* tab_h = stg.take<float2>(tabs.size() > 0 ? tabs.size() : 1);
  if (!tabs.empty()) std::memcpy(tab_h, tabs.data(), tabs.size() * sizeof(float2));
  r->stitch_desc.ensure(p.n_desc * sizeof(fragk::StitchChunk));
  r->stitch_tab.ensure(std::max<size_t>(tabs.size(), 1) * sizeof(float2));
  check_cuda(cudaMemcpyAsync(r->stitch_desc.p, desc, p.n_desc * sizeof(fragk::StitchChunk), cudaMemcpyHostToDevice,
                             s),
             "stitch desc");
  if (!tabs.empty())
    check_cuda(cudaMemcpyAsync(r->stitch_tab.p, tab_h, tabs.size() * sizeof(float2), cudaMemcpyHostToDevice, s),
               "stitch tab");
  for (int i = 0; i < p.n_desc; ++i) p.bytes += (r->vshared ? 2.0 : 4.0) * c.layers * desc[i].n_tok * kvc * sizeof(bf16);
  return p;
}

StitchPlan stitch_prepare(Engine* e, Result* r, cudaStream_t s, Stage& stg, const SysKV* sys,
                          const std::vector<Record*>& recs, int S) {
  return stitch_prepare_parts(e, r, s, stg, {StitchPart{sys, &recs, S, 0}});
}

// ---- shared V pages
// A request reads V in place only from records in this device's memory (an
// attached peer's or IPC-imported pages would be re-read over NVLink by every
// layer's attention: those requests keep the one-pass copy of K1).
bool records_local(const Engine* e, const std::vector<Record*>& recs) {
  for (const Record* rec : recs) {
    if (rec->tier == FRAG_TIER_PEER || rec->ipc_mapped) return false;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, rec->kv.p) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    if (at.device != e->device) return false;
  }
  return true;
}

// One sequence of a shared-V request: its V segments (KV_S, then the records
// in prompt order), cache rows and the exclusive slots of its fresh rows.
struct VPart {
  const SysKV* sys;
  const std::vector<Record*>* recs;
  int S, base, T, nq, k;
  int plan_off;      // GEMM row of its first critical row (= its exclusive slot)
  int tail_slot_q;   // exclusive slot of its first question row in the question pass
  int tail_slot_s;   // ... in the sparse pass (and decode)
};

// Host prep: segment table with each segment's TMA map, per-sequence plan
// slices and the two plan-build argument sets ([0, B): question pass, no
// critical rows; [B, 2B): sparse pass, the selected rows in plan_rows), the
// exclusive region (vx_rows slots per layer) and references that keep the
// records' pages alive for as long as this result reads them.
void vshared_prepare(Engine* e, Result* r, cudaStream_t s, Stage& stg, const std::vector<VPart>& parts, int n_rows,
                     int vx_rows) {
  const auto& c = e->cfg;
  const uint64_t kvc = (uint64_t)c.n_kv_heads * c.head_dim;
  const int B = (int)parts.size();
  int n_seg = 0;
  for (const auto& pt : parts) n_seg += (pt.sys && pt.sys->n > 0 ? 1 : 0) + (int)pt.recs->size();
  const int tiles = (n_rows + 127) / 128;
  r->vseg.ensure((size_t)std::max(n_seg, 1) * sizeof(fragk::VSeg));
  r->vplan_tile.ensure((size_t)B * (tiles + 1) * sizeof(int));
  r->vplan_prim.ensure((size_t)B * tiles * sizeof(int2));
  r->vplan_ent.ensure((size_t)B * n_rows * sizeof(unsigned long long));
  r->vplan_args.ensure((size_t)2 * B * sizeof(fragk::VPlanArgs));
  r->vx_rows = vx_rows;
  r->vx.ensure((size_t)c.layers * vx_rows * kvc * sizeof(bf16));
  auto* segs = stg.take<fragk::VSeg>(std::max(n_seg, 1));
  auto* args = stg.take<fragk::VPlanArgs>(2 * B);
  // exclusive slots as one tensor (rows = slots), box (64, 1, 1): patched rows
  // [0]: box rows 1 (one patched row), [1]: box rows 32 (a staged run of fresh rows)
  auto* xmap = stg.take<CUtensorMap>(2);
  r->vx_map.ensure(2 * sizeof(CUtensorMap));
  for (int i = 0; i < 2; ++i)
    if (!fragk::make_tmap_3d(&xmap[i], r->vx.p, kvc, (uint64_t)vx_rows, (uint64_t)c.layers, kvc,
                             (uint64_t)vx_rows * kvc, 64, i ? 32 : 1, 1))
      fail(FRAG_E_CUDA, "shared V: tensor map encoding failed");
  check_cuda(cudaMemcpyAsync(r->vx_map.p, xmap, 2 * sizeof(CUtensorMap), cudaMemcpyHostToDevice, s), "V slot maps");
  r->vseq.clear();
  r->vrefs.clear();
  r->vseg_max_rows = 0;
  r->vseg_rows = 0;
  int si = 0, cur_base = 0;
  auto add = [&](const bf16* v, int n, int row0) {
    fragk::VSeg& g = segs[si++];
    std::memset(&g, 0, sizeof(g));
    // V [L][n][Hkv*dh] as (Hkv*dh, n, L); box (64 cols, 128 rows, 1 layer)
    if (!fragk::make_tmap_3d(&g.tmap, v, kvc, (uint64_t)n, (uint64_t)c.layers, kvc, (uint64_t)n * kvc, 64, 128, 1) ||
        !fragk::make_tmap_3d(&g.tmap1, v, kvc, (uint64_t)n, (uint64_t)c.layers, kvc, (uint64_t)n * kvc, 64, 1, 1))
      fail(FRAG_E_CUDA, "shared V: tensor map encoding failed");
    g.v = v;
    g.row0 = row0;
    g.n = n;
    g.base = cur_base;
    r->vseg_max_rows = std::max(r->vseg_max_rows, n);
    r->vseg_rows += n;
  };
  fragk::VSeg* seg_dev = r->vseg.as<fragk::VSeg>();
  for (int b = 0; b < B; ++b) {
    const VPart& pt = parts[b];
    Result::VSeq q{};
    q.seg0 = si;
    cur_base = pt.base;
    if (pt.sys && pt.sys->n > 0) add(pt.sys->kv.as<bf16>() + (size_t)c.layers * pt.sys->n * kvc, pt.sys->n, 0);
    int row = pt.S;
    for (Record* rec : *pt.recs) {
      add(rec->v(), rec->n_tok, row);
      row += rec->n_tok;
      r->vrefs.push_back(rec->shared_from_this());
    }
    q.n_seg = si - q.seg0;
    q.n_rows = n_rows;
    q.vt_off = b * (tiles + 1);
    q.vp_off = b * tiles;
    q.ve_off = b * n_rows;
    q.base = pt.base;
    q.T = pt.T;
    q.tail_row0 = pt.T - pt.nq;
    q.tail_slot_q = pt.tail_slot_q;
    q.tail_slot_s = pt.tail_slot_s;
    r->vseq.push_back(q);
    for (int w = 0; w < 2; ++w) {
      fragk::VPlanArgs& a = args[w * B + b];
      a.segs = seg_dev + q.seg0;
      a.n_seg = q.n_seg;
      a.crit = w ? r->plan_rows.as<int>() + pt.plan_off : nullptr;
      a.n_crit = w ? pt.k : 0;
      a.row_base = pt.base;
      a.crit_slot0 = pt.plan_off;
      a.tail_row0 = q.tail_row0;
      a.n_rows = n_rows;
      a.vtile = r->vplan_tile.as<int>() + q.vt_off;
      a.vprim = r->vplan_prim.as<int2>() + q.vp_off;
      a.vent = r->vplan_ent.as<unsigned long long>() + q.ve_off;
    }
  }
  r->vseg_n = n_seg;
  check_cuda(cudaMemcpyAsync(r->vseg.p, segs, (size_t)n_seg * sizeof(fragk::VSeg), cudaMemcpyHostToDevice, s),
             "V segments");
  check_cuda(cudaMemcpyAsync(r->vplan_args.p, args, (size_t)2 * B * sizeof(fragk::VPlanArgs), cudaMemcpyHostToDevice,
                             s),
             "V plan args");
}

// Build the patch plans (which = 0: question pass, 1: sparse pass) on the
// request stream (part of the captured body).
void vplan_launch(Engine* e, Result* r, cudaStream_t s, int which) {
  if (!r->vshared || r->vseq.empty()) return;
  const int B = (int)r->vseq.size();
  int max_segs = 0;
  for (const auto& q : r->vseq) max_segs = std::max(max_segs, q.n_seg);
  Scoped sc(e->prof, s, KC_SELECT, 0, 0);
  const int rc = fragk::vpatch_plan(r->vplan_args.as<fragk::VPlanArgs>() + which * B, B, r->vseq[0].n_rows, max_segs, s);
  if (rc < 0) fail(FRAG_E_CUDA, "shared V plan launch failed");
  sc.launched(rc);
}

void stitch_launch(Engine* e, Result* r, cudaStream_t s, const StitchPlan& p, int l0 = 0, int l1 = -1) {
  if (p.n_desc == 0) return;
  const auto& c = e->cfg;
  if (l1 < 0) l1 = c.layers;
  Scoped sc(e->prof, s, KC_STITCH, 0, p.bytes * (l1 - l0) / c.layers);
  // shared V pages: K only (V stays in the records)
  sc.launched(fragk::rope_shift_assemble(r->stitch_desc.as<fragk::StitchChunk>(), p.n_desc, p.max_rows,
                                         r->stitch_tab.as<float2>(), r->k_fused.as<bf16>(),
                                         r->vshared ? nullptr : r->v_fused.as<bf16>(), l1 - l0, r->max_tokens,
                                         c.n_kv_heads, c.head_dim, s, l0));
  peek("stitch");
}

// K1 layer by layer on the result's side stream, forked from `s`; layer l's
// completion is r->layer_ev[l]. The question pass (on `s`) waits for layer l
// only before its layer-l attention, so the HBM-bound stitch streams under the
// latency-bound M = |Q| weight stream instead of in front of it.
// Off by default (FRAG_STITCH_OVERLAP=1 enables it): measured on B200 the
// request is power-capped end to end (sw_power_cap, ~1.45 GHz), so hiding the
// 0.7 ms stitch under the question pass moved no TTFT (45.9 vs 45.8 ms), while
// 32 per-layer launches run the HBM stream at half the bandwidth of the single
// launch (3.0 vs 5.9 TB/s) -- kept as an option for uncapped parts.
bool stitch_overlap_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("FRAG_STITCH_OVERLAP");
    return v && v[0] == '1';
  }();
  return on;
}
// r = 0 fast path (one full pass over the question rows instead of question
// pass + sparse pass); FRAG_R0_FAST=0 restores the two passes (A/B, tests)
bool r0_fast_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("FRAG_R0_FAST");
    return !(v && v[0] == '0');
  }();
  return on;
}
void stitch_fork(Engine* e, Result* r, cudaStream_t s, const StitchPlan& p) {
  const int L = e->cfg.layers;
  if (!r->side) check_cuda(cudaStreamCreateWithFlags(&r->side, cudaStreamNonBlocking), "side stream");
  if (!r->fork_ev) check_cuda(cudaEventCreateWithFlags(&r->fork_ev, cudaEventDisableTiming), "fork event");
  while ((int)r->layer_ev.size() < L) {
    cudaEvent_t ev;
    check_cuda(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "layer event");
    r->layer_ev.push_back(ev);
  }
  check_cuda(cudaEventRecord(r->fork_ev, s), "fork");
  check_cuda(cudaStreamWaitEvent(r->side, r->fork_ev, 0), "fork wait");
  for (int l = 0; l < L; ++l) {
    stitch_launch(e, r, r->side, p, l, l + 1);
    check_cuda(cudaEventRecord(r->layer_ev[l], r->side), "layer stitched");
  }
}

void stitch(Engine* e, Result* r, cudaStream_t s, Stage& stg, const SysKV* sys, const std::vector<Record*>& recs,
            int S) {
  stitch_launch(e, r, s, stitch_prepare(e, r, s, stg, sys, recs, S));
}

// Replay the request body from a CUDA graph when its shape was seen before
// and no device buffer was (re)allocated since the capture; otherwise run it
// eagerly (first sighting, per-stage timing, or profiling).
template <class Body>
void run_graphed(Result* r, cudaStream_t s, bool graphable, const GraphKey& key, Body&& body) {
  static const bool graphs_env = [] {  // FRAG_GRAPHS=0: always launch eagerly
    const char* v = std::getenv("FRAG_GRAPHS");
    return !(v && v[0] == '0');
  }();
  if (!graphable || !graphs_env) {
    body(s);
    return;
  }
  const uint64_t epoch = g_alloc_epoch.load();
  auto it = r->graphs.find(key);
  if (it != r->graphs.end() && it->second.epoch == epoch) {
    g_launches += it->second.launches;
    check_cuda(cudaGraphLaunch(it->second.exec, s), "cudaGraphLaunch");
    return;
  }
  if (it != r->graphs.end()) {
    cudaGraphExecDestroy(it->second.exec);
    r->graphs.erase(it);
  }
  if (r->graphs.size() >= 64) {  // bound the cache: many distinct shapes -> start over
    for (auto& g : r->graphs) cudaGraphExecDestroy(g.second.exec);
    r->graphs.clear();
    r->seen.clear();
  }
  if (!r->seen.count(key)) {  // first sighting: run eagerly so every buffer reaches its final size
    body(s);
    r->seen.insert(key);
    return;
  }
  // capture on a private stream: the caller's may be the legacy default
  // stream, which cannot be captured; the graph is then launched on `s`
  if (!r->cap_stream) check_cuda(cudaStreamCreateWithFlags(&r->cap_stream, cudaStreamNonBlocking), "capture stream");
  cudaStream_t cs = r->cap_stream;
  cudaGraph_t g = nullptr;
  const uint64_t l0 = g_launches.load();
  check_cuda(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal), "begin capture");
  try {
    body(cs);
  } catch (...) {
    cudaStreamEndCapture(cs, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  check_cuda(cudaStreamEndCapture(cs, &g), "end capture");
  GraphEntry ent;
  ent.launches = g_launches.load() - l0;
  g_launches -= ent.launches;  // counted when the graph is launched
  cudaError_t err = cudaGraphInstantiate(&ent.exec, g, 0);
  cudaGraphDestroy(g);
  check_cuda(err, "cudaGraphInstantiate");
  ent.epoch = g_alloc_epoch.load();
  r->graphs.emplace(key, ent);
  g_launches += ent.launches;
  check_cuda(cudaGraphLaunch(ent.exec, s), "cudaGraphLaunch");
}

Result* scratch_for(Engine* e, int tokens) {
  if (!e->scratch || e->scratch->max_tokens < tokens) {
    e->scratch = std::make_unique<Result>();
    result_init(e->scratch.get(), e, std::max(tokens, 256));
  }
  use_private_v(e->scratch.get());
  return e->scratch.get();
}

// KV_S of the system prompt, computed once per token list.
SysKV* get_sys_kv(Engine* e, const int32_t* sys, int n_sys, cudaStream_t s) {
  if (n_sys <= 0) return nullptr;
  std::vector<int32_t> key(sys, sys + n_sys);
  std::lock_guard<std::mutex> g(e->mu);
  auto it = e->sys_cache.find(key);
  if (it != e->sys_cache.end()) return it->second.get();
  const auto& c = e->cfg;
  for (int i = 0; i < n_sys; ++i)
    if (sys[i] < 0 || sys[i] >= c.vocab) fail(FRAG_E_CONTRACT, "system token out of vocabulary");
  Result* r = scratch_for(e, n_sys);
  std::vector<int> rows(n_sys);
  for (int i = 0; i < n_sys; ++i) rows[i] = i;
  check_cuda(cudaMemcpyAsync(r->plan_rows.p, rows.data(), n_sys * sizeof(int), cudaMemcpyHostToDevice, s), "sys rows");
  check_cuda(cudaMemcpyAsync(r->plan_tok.p, sys, n_sys * sizeof(int), cudaMemcpyHostToDevice, s), "sys tok");
  run_rows(e, r, s, n_sys, n_sys, PASS_KV_ONLY, nullptr, 0);
  auto kv = std::make_unique<SysKV>();
  kv->n = n_sys;
  const size_t kvc = (size_t)c.n_kv_heads * c.head_dim;
  const size_t w = (size_t)n_sys * kvc * sizeof(bf16), pitch = (size_t)r->max_tokens * kvc * sizeof(bf16);
  kv->kv.alloc(2 * (size_t)c.layers * w);
  check_cuda(cudaMemcpy2DAsync(kv->kv.p, w, r->k_fused.p, pitch, w, c.layers, cudaMemcpyDeviceToDevice, s), "sysK");
  check_cuda(cudaMemcpy2DAsync(kv->kv.as<char>() + c.layers * w, w, r->v_fused.p, pitch, w, c.layers,
                               cudaMemcpyDeviceToDevice, s),
             "sysV");
  sync_checked(e, r, s, "system prompt prefill");
  SysKV* out = kv.get();
  e->sys_cache.emplace(std::move(key), std::move(kv));
  return out;
}

// ---- kv_deviation / select_cacheblend (Eq. 7-8)
// The Full-Attention rows of the first Ld layers are computed in place over the
// chunk rows [S, S+N) of the result's fused cache (system rows are KV_S in
// both modes, Eq. 4), after the stitched Full-Reuse rows of those layers were
// saved to r->fr_save; the deviation kernel compares the two, then the saved
// rows are copied back so the cache is Full Reuse again for the sparse pass.
void fr_copy(Engine* e, Result* r, cudaStream_t s, int S, int N, int Ld, bool restore) {
  const auto& c = e->cfg;
  const size_t kvc = (size_t)c.n_kv_heads * c.head_dim;
  const size_t w = (size_t)N * kvc * sizeof(bf16), pitch = (size_t)r->max_tokens * kvc * sizeof(bf16);
  char* kf = r->k_fused.as<char>() + (size_t)S * kvc * sizeof(bf16);
  char* vf = r->v_fused.as<char>() + (size_t)S * kvc * sizeof(bf16);
  char* ks = r->fr_save.as<char>();
  char* vs = ks + (size_t)Ld * w;
  const cudaMemcpyKind kd = cudaMemcpyDeviceToDevice;
  if (!restore) {
    check_cuda(cudaMemcpy2DAsync(ks, w, kf, pitch, w, Ld, kd, s), "save FR K");
    check_cuda(cudaMemcpy2DAsync(vs, w, vf, pitch, w, Ld, kd, s), "save FR V");
  } else {
    check_cuda(cudaMemcpy2DAsync(kf, pitch, ks, w, w, Ld, kd, s), "restore FR K");
    check_cuda(cudaMemcpy2DAsync(vf, pitch, vs, w, w, Ld, kd, s), "restore FR V");
  }
}

// FA pass over the chunk rows (plan rows S.. / chunk tokens must be on the
// device) + the deviation kernel. dev: [N][Ld][2] or null; sel: [N] or null.
void deviation_body(Engine* e, Result* r, cudaStream_t s, int S, int N, int Ld, float* dev, float* sel,
                    int sel_comp) {
  const auto& c = e->cfg;
  const size_t kvc = (size_t)c.n_kv_heads * c.head_dim;
  fr_copy(e, r, s, S, N, Ld, false);
  run_rows(e, r, s, N, S + N, PASS_KV_ONLY, nullptr, 0, Ld);
  fragk::DeviationArgs a{};
  a.k_fa = r->k_fused.as<bf16>() + (size_t)S * kvc;
  a.v_fa = r->v_fused.as<bf16>() + (size_t)S * kvc;
  a.fa_layer_stride = (size_t)r->max_tokens * kvc;
  a.k_fr = r->fr_save.as<bf16>();
  a.v_fr = r->fr_save.as<bf16>() + (size_t)Ld * N * kvc;
  a.fr_layer_stride = (size_t)N * kvc;
  a.n_rows = N;
  a.n_layers = Ld;
  a.width = (int)kvc;
  a.dev = dev;
  a.sel_scores = sel;
  a.sel_layer = Ld - 1;
  a.sel_comp = sel_comp;
  {
    Scoped sc(e->prof, s, KC_SELECT, 0, 4.0 * N * Ld * kvc * sizeof(bf16));
    sc.launched(fragk::kv_deviation(a, s));
  }
  fr_copy(e, r, s, S, N, Ld, true);
  peek("kv_deviation");
}

void ev_record(Result* r, bool on, int i, cudaStream_t s) {
  if (on) cudaEventRecord(r->ev[i], s);
}

void logits_d2h(Result* r, cudaStream_t s) {
  if (r->logits_on_device || r->logit_rows == 0) return;
  const size_t n = (size_t)r->logit_rows * r->eng->cfg.vocab;
  check_cuda(cudaMemcpyAsync(r->logits_host.p, r->logits.p, n * sizeof(float), cudaMemcpyDeviceToHost, s),
             "logits D2H");
}

void finish(Result* r, bool timing, cudaStream_t s) {
  Engine* e = r->eng;
  ev_record(r, timing, 6, s);
  r->last_stream = s;
  sync_checked(e, r, s, "reprocess");
  e->prof.collect();
  r->timing_valid = timing;
  if (timing) {
    float t[6] = {};
    for (int i = 0; i < 6; ++i) cudaEventElapsedTime(&t[i], r->ev[i], r->ev[i + 1]);
    r->timing.stitch_ms = t[0];
    r->timing.question_ms = t[1];
    r->timing.select_ms = t[2];
    r->timing.sparse_ms = t[3];
    r->timing.lm_head_ms = t[4] + t[5];
    cudaEventElapsedTime(&r->timing.total_ms, r->ev[0], r->ev[6]);
  }
}

}  // namespace

// ---------------------------------------------------------------- reprocess
// Host prep (record fetch, RoPE/stitch tables, staging + H2D of the small
// per-request inputs) runs every call; the device body (K1 -> question pass ->
// K9/K10 -> sparse pass -> lm_head -> logits D2H) is captured once per request
// shape into a CUDA graph and replayed, so ~500 launches cost one.
void reprocess(Engine* e, Store* st, const int32_t* sys, int n_sys, const int32_t* q_tokens, int n_q,
               bool q_on_device, const frag_chunk_id* ids, int n_chunks, float ratio,
               const frag_reprocess_opts* o, cudaStream_t s, Result* r) {
  std::lock_guard<std::recursive_mutex> gpu_lock(device_mutex(e->device));
  const auto& c = e->cfg;
  const auto t_entry = std::chrono::steady_clock::now();
  if (!r || r->eng != e) fail(FRAG_E_CONTRACT, "result does not belong to this engine");
  if (!st) fail(FRAG_E_CONTRACT, "store is null");
  if (st->device != e->device) fail(FRAG_E_CONTRACT, "store and engine are on different devices");
  if (n_q < 1) fail(FRAG_E_CONTRACT, "question must have at least one token");
  if (n_sys < 0 || n_chunks < 0) fail(FRAG_E_CONTRACT, "negative length");
  if (!(ratio >= 0.f && ratio <= 1.f)) fail(FRAG_E_CONTRACT, "recompute_ratio must lie in [0, 1]");
  if (n_chunks > 0 && !ids) fail(FRAG_E_CONTRACT, "chunk_ids is null");
  DeviceGuard dg(e->device);
  const bool timing = o && o->timing;
  if (!q_on_device)
    for (int i = 0; i < n_q; ++i)
      if (q_tokens[i] < 0 || q_tokens[i] >= c.vocab) fail(FRAG_E_CONTRACT, "question token out of vocabulary");

  PinGuard pins{st, {}};
  std::vector<Record*> recs;
  for (int i = 0; i < n_chunks; ++i) {
    Record* rec = store_try_fetch(st, ids[i]);  // heat++, pin
    if (!rec) {
      const int32_t* ft = (o && o->fallback_tokens) ? o->fallback_tokens[i] : nullptr;
      const int fl = (o && o->fallback_lens) ? o->fallback_lens[i] : 0;
      if (!ft || fl < 1)
        fail(FRAG_E_STORE, "missing chunk record " + std::to_string(i) +
                               " (SPEC.md:287); stitch_full_reuse needs every chunk matched -- pass its tokens in "
                               "frag_reprocess_opts.fallback_tokens for an on-the-fly isolated prefill (SPEC.md:403)");
      // flag-gated fallback: isolated prefill of the chunk (Eq. 5) into the store
      frag_chunk_id got;
      hash_tokens(ft, fl, 0, &got);
      if (std::memcmp(got.bytes, ids[i].bytes, 16) != 0)
        fail(FRAG_E_CONTRACT, "fallback tokens of chunk " + std::to_string(i) + " do not hash to its chunk id");
      preprocess_isolated(e, st, sys, n_sys, ft, fl, false, &got);
      rec = store_fetch(st, ids[i]);
    }
    recs.push_back(rec);
    pins.ids.push_back(ids[i]);
  }
  const int S = n_sys;
  int N = 0;
  for (Record* rec : recs) N += rec->n_tok;
  const int T = S + N + n_q;
  if (T > r->max_tokens)
    fail(FRAG_E_CONTRACT, "prompt of " + std::to_string(T) + " tokens exceeds the result capacity " +
                              std::to_string(r->max_tokens));
  const bool inject = o && o->inject_crit;
  int k = (int)std::floor((double)ratio * (double)N + 0.5);  // |C_idx| = round(r * sum|C|)
  if (inject) {
    k = o->n_inject;
    if (k < 0 || k > N) fail(FRAG_E_CONTRACT, "injected critical set larger than the chunk tokens");
    for (int i = 0; i < k; ++i) {
      const int p = o->inject_crit[i];
      if (p < S + 1 || p > S + N) fail(FRAG_E_CONTRACT, "critical position outside the chunk range (SPEC.md:391)");
      if (i > 0 && p <= o->inject_crit[i - 1]) fail(FRAG_E_CONTRACT, "critical positions must be strictly increasing");
    }
    if (q_on_device) fail(FRAG_E_CONTRACT, "selection injection requires host question tokens");
  }
  const int M = k + n_q;
  const int selector = o ? o->selector : FRAG_SELECT_QUERY_GUIDED;
  if (selector != FRAG_SELECT_QUERY_GUIDED && selector != FRAG_SELECT_CACHEBLEND)
    fail(FRAG_E_CONTRACT, "unknown selector");
  const int dev_layer = (o && o->deviation_layer > 0) ? o->deviation_layer : 2;
  const int dev_comp = o ? o->deviation_component : FRAG_DEV_K;
  if (selector == FRAG_SELECT_CACHEBLEND) {
    if (dev_layer > c.layers) fail(FRAG_E_CONTRACT, "deviation_layer exceeds the model depth");
    if (dev_comp < FRAG_DEV_K || dev_comp > FRAG_DEV_KV) fail(FRAG_E_CONTRACT, "unknown deviation component");
  }
  // select_cacheblend replaces the question pass + K9
  const bool cacheblend = selector == FRAG_SELECT_CACHEBLEND && !inject && N > 0;
  // shared V pages: the default for query-guided / injected requests over this
  // device's records with at most half of the chunk rows recomputed (the
  // attention patches every fresh row into its V tiles)
  const bool vsh = !cacheblend && N > 0 && 2L * k <= N && shared_v_enabled() &&
                   fragk::attn_shared_v_supported(c.head_dim) &&
                   fragk::vpatch_plan_fits(r->max_tokens, n_chunks + 1) && records_local(e, recs);
  if (vsh) {
    if (!r->vshared) r->v_fused.release();  // an earlier request's private V (a read-back view is kept)
    r->vshared = true;
    r->v_materialized = false;
    r->v_tail_row0 = T - n_q;  // question rows (and decoded tokens) -> slots k, k+1, ...
    r->v_tail_slot0 = k;
  } else {
    use_private_v(r);
  }
  e->ensure_rope(T);
  SysKV* skv = get_sys_kv(e, sys, n_sys, s);
  if (cacheblend)
    r->fr_save.ensure((size_t)2 * dev_layer * N * c.n_kv_heads * c.head_dim * sizeof(bf16));

  r->T = T;
  r->rows_per_seq = 0;
  r->batch.clear();
  r->S = S;
  r->N = N;
  r->nq = n_q;
  r->k_sel = k;
  r->M = M;
  const bool all_logits = o && o->all_logits;
  const bool raw = o && o->raw_scores;
  r->logit_rows = all_logits ? n_q : 1;
  r->logits_on_device = o && o->logits_on_device;

  // ---- host prep: everything that depends on this request's chunks / tokens
  r->staging.ensure(64 * 1024 + (size_t)(n_chunks + 2) * (64 + c.head_dim * 4 + sizeof(fragk::VSeg)) +
                    (size_t)(4 * T + 4 * M + 4 * n_q) * 4);
  Stage stg(r->staging);
  // injected plan first: the captured body copies from these staging slots,
  // so their offsets must depend only on the graph key
  int* inj_rows = inject ? stg.take<int>(M) : nullptr;
  int* inj_tok = inject ? stg.take<int>(M) : nullptr;
  int* cb_rows = cacheblend ? stg.take<int>(N) : nullptr;  // FA-pass plan rows S..S+N-1 (copied in the body)
  if (cacheblend)
    for (int i = 0; i < N; ++i) cb_rows[i] = S + i;
  StitchPlan sp = stitch_prepare(e, r, s, stg, skv, recs, S);
  if (vsh) vshared_prepare(e, r, s, stg, {VPart{skv, &recs, S, 0, T, n_q, k, 0, k, k}}, r->max_tokens,
                           k + r->max_tokens - (T - n_q));
  {
    int off = 0;  // chunk token ids in prompt order (the recompute gather, K2)
    for (Record* rec : recs) {
      check_cuda(cudaMemcpyAsync(r->chunk_tok.as<int>() + off, rec->tok.p, rec->n_tok * sizeof(int),
                                 cudaMemcpyDeviceToDevice, s),
                 "chunk tokens");
      off += rec->n_tok;
    }
  }
  if (q_on_device) {
    check_cuda(cudaMemcpyAsync(r->q_tok.p, q_tokens, n_q * sizeof(int), cudaMemcpyDeviceToDevice, s), "q tok");
  } else {
    int* qh = stg.take<int>(n_q);
    std::memcpy(qh, q_tokens, n_q * sizeof(int));
    check_cuda(cudaMemcpyAsync(r->q_tok.p, qh, n_q * sizeof(int), cudaMemcpyHostToDevice, s), "q tok");
  }
  {
    int* rows_h = stg.take<int>(n_q);  // question-pass plan: the last n_q rows
    for (int i = 0; i < n_q; ++i) rows_h[i] = T - n_q + i;
    check_cuda(cudaMemcpyAsync(r->plan_rows.p, rows_h, n_q * sizeof(int), cudaMemcpyHostToDevice, s), "q rows");
    check_cuda(cudaMemcpyAsync(r->plan_tok.p, r->q_tok.p, n_q * sizeof(int), cudaMemcpyDeviceToDevice, s), "q plan");
  }
  if (inject) {  // written now, copied inside the body after the question pass
    for (int i = 0; i < k; ++i) {
      const int row = o->inject_crit[i] - 1;
      inj_rows[i] = row;
      int j = row - S, t = 0;
      for (Record* rec : recs) {
        if (j < rec->n_tok) {
          t = rec->tok_host[j];
          break;
        }
        j -= rec->n_tok;
      }
      inj_tok[i] = t;
    }
    for (int i = 0; i < n_q; ++i) {
      inj_rows[k + i] = T - n_q + i;
      inj_tok[k + i] = q_tokens[i];
    }
  }
  {
    int* map_h = stg.take<int>(r->logit_rows);
    if (all_logits)
      for (int i = 0; i < n_q; ++i) map_h[i] = k + i;
    else
      map_h[0] = M - 1;
    check_cuda(cudaMemcpyAsync(r->row_map.p, map_h, r->logit_rows * sizeof(int), cudaMemcpyHostToDevice, s), "map");
  }
  if (N > 0 && !inject) {
    r->part_ms.ensure((size_t)((N + 31) / 32) * n_q * c.n_heads * sizeof(float2));
    r->row_ms.ensure((size_t)n_q * c.n_heads * sizeof(float2));
    r->score_col.ensure(fragk::score_col_part_elems(n_q, c.n_heads, c.n_kv_heads, N) * sizeof(float));
    r->score_q.ensure(fragk::score_q_split_elems(n_q, c.n_heads, c.n_kv_heads, c.head_dim) * sizeof(bf16));
  }
  r->lm_x.ensure((size_t)r->logit_rows * c.d_model * sizeof(bf16));
  r->logits.ensure((size_t)r->logit_rows * c.vocab * sizeof(float));
  if (!r->logits_on_device) r->logits_host.ensure((size_t)r->logit_rows * c.vocab * sizeof(float));

  // ---- device body
  const bool full_reuse = k == 0 && !cacheblend && !inject && r0_fast_enabled();
  // K1 overlapped with the question pass (the stitch_ms stage is then ~0 and
  // question_ms covers both); CacheBlend's 2-layer FA pass needs it up front
  const bool overlap = !cacheblend && sp.n_desc > 0 && c.layers > 1 && stitch_overlap_enabled();
  auto body = [&](cudaStream_t bs) {
    ev_record(r, timing, 0, bs);
    if (overlap)
      stitch_fork(e, r, bs, sp);  // K1 per layer on the side stream
    else
      stitch_launch(e, r, bs, sp);  // K1: stitch_full_reuse
    ev_record(r, timing, 1, bs);
    vplan_launch(e, r, bs, 0);  // shared V: patch plan without critical rows (question pass)
    if (full_reuse) {
      // r = 0 (Full Reuse): the plan is exactly the
      // question rows, so the sparse pass would recompute what the question
      // pass computes; one full pass over those rows gives the logits (and
      // q_final from its last QKV) -- bit-identical to question pass + sparse pass
      r->q_final_in_full = true;
      run_rows(e, r, bs, n_q, T, PASS_FULL, nullptr, 0, 0, overlap ? r->layer_ev.data() : nullptr, nullptr,
               r->logit_rows);
      r->q_final_in_full = false;
      if (overlap) check_cuda(cudaStreamWaitEvent(bs, r->layer_ev[c.layers - 1], 0), "join stitch");
      ev_record(r, timing, 2, bs);
      ev_record(r, timing, 3, bs);
    } else {
    // question pass: last_layer_query_states against the stitched cache
    if (!cacheblend) run_rows(e, r, bs, n_q, T, PASS_QUESTION, nullptr, 0, 0, overlap ? r->layer_ev.data() : nullptr);
    if (overlap)  // join: every stitched layer (the last one feeds the selection keys)
      check_cuda(cudaStreamWaitEvent(bs, r->layer_ev[c.layers - 1], 0), "join stitch");
    ev_record(r, timing, 2, bs);
    // select_query_guided (K9 + K10) -> QIndexPlan on device
    if (cacheblend) {
      // select_cacheblend: Delta_KV[:, dev_layer, comp] between Full Attention and
      // Full Reuse over cat(S, chunks) (Eq. 7-8), then the same top-k plan (K10)
      check_cuda(cudaMemcpyAsync(r->plan_rows.p, cb_rows, N * sizeof(int), cudaMemcpyHostToDevice, bs), "fa rows");
      check_cuda(cudaMemcpyAsync(r->plan_tok.p, r->chunk_tok.p, N * sizeof(int), cudaMemcpyDeviceToDevice, bs),
                 "fa tok");
      deviation_body(e, r, bs, S, N, dev_layer, nullptr, r->scores.as<float>(), dev_comp);
      Scoped sc(e->prof, bs, KC_SELECT, 0, 4.0 * N * 6);
      sc.launched(fragk::topk_plan(r->scores.as<float>(), N, k, S, r->chunk_tok.as<int>(), r->q_tok.as<int>(), n_q,
                                   T - n_q, r->plan_rows.as<int>(), r->plan_tok.as<int>(), bs));
    } else if (inject) {
      check_cuda(cudaMemcpyAsync(r->plan_rows.p, inj_rows, M * sizeof(int), cudaMemcpyHostToDevice, bs), "plan rows");
      check_cuda(cudaMemcpyAsync(r->plan_tok.p, inj_tok, M * sizeof(int), cudaMemcpyHostToDevice, bs), "plan tok");
    } else {
      if (N > 0) {
        fragk::ScoreArgs a{};
        a.q = r->q_final.as<float>();
        a.k = r->k_fused.as<bf16>() + (size_t)(c.layers - 1) * r->max_tokens * c.n_kv_heads * c.head_dim;
        a.nq = n_q;
        a.Hq = c.n_heads;
        a.Hkv = c.n_kv_heads;
        a.dh = c.head_dim;
        a.key_row0 = S;
        a.n_keys = N;
        a.scale = 1.0f / std::sqrt((float)c.head_dim);
        a.part_ms = r->part_ms.as<float2>();
        a.row_ms = r->row_ms.as<float2>();
        a.scores = r->scores.as<float>();
        a.raw = raw;
        a.col_part = r->score_col.as<float>();
        a.q_split = r->score_q.as<bf16>();
        Scoped sc(e->prof, bs, KC_SELECT, 4.0 * n_q * c.n_heads * (double)N * c.head_dim,
                  2.0 * N * (double)c.n_kv_heads * c.head_dim * 2);
        sc.launched(fragk::qg_score(a, bs));
      }
      Scoped sc(e->prof, bs, KC_SELECT, 0, 4.0 * N * 6);
      sc.launched(fragk::topk_plan(r->scores.as<float>(), N, k, S, r->chunk_tok.as<int>(), r->q_tok.as<int>(), n_q,
                                   T - n_q, r->plan_rows.as<int>(), r->plan_tok.as<int>(), bs));
    }
    peek("select");
    vplan_launch(e, r, bs, 1);  // shared V: + the critical rows' exclusive slots
    ev_record(r, timing, 3, bs);
    // sparse_prefill (Eq. 9) to the first-token logits
    run_rows(e, r, bs, M, T, PASS_FULL, nullptr, 0, 0, nullptr, nullptr, r->logit_rows);
    }
    ev_record(r, timing, 4, bs);
    {
      // final norm + lm_head on the logit rows (K3 + K11)
      const int d = c.d_model;
      {
        Scoped sc(e->prof, bs, KC_NORM, 0, (double)r->logit_rows * d * 6);
        fragk::rmsnorm(r->h.as<float>(), r->logit_rows, d, e->final_norm, c.norm_eps, r->lm_x.as<bf16>(), bs,
                       r->row_map.as<int>());
        sc.launched(1);
      }
      fragk::EpiParams ep;
      ep.ws = r->gemm_ws.as<float>();
      ep.ws_bytes = r->gemm_ws.bytes;
      ep.counters = r->gemm_cnt.as<int>();
      ep.counters_cap = gemm_counter_cap(r);
      ep.out_f32 = r->logits.as<float>();
      ep.ldo = c.vocab;
      Scoped sc(e->prof, bs, gemm_class(r->logit_rows), 2.0 * r->logit_rows * (double)c.vocab * d, 2.0 * c.vocab * (double)d);
      sc.launched(fragk::gemm_bf16_tc(r->lm_x.as<bf16>(), e->lm_head, r->logit_rows, c.vocab, d,
                                      fragk::EPI_STORE_F32, ep, bs));
    }
    peek("lm_head");
    ev_record(r, timing, 5, bs);
    logits_d2h(r, bs);
  };

  const bool graphable = !timing && !e->prof.on;
  GraphKey key{T, S, N, n_q, k, (int)inject, (int)all_logits, (int)raw, (int)r->logits_on_device, sp.n_desc,
               sp.max_rows,
               (cacheblend ? 1 + dev_layer * 4 + dev_comp : 0) + (overlap ? 1000 : 0) + (full_reuse ? 2000 : 0) +
                   (vsh ? 4000 : 0),
               (uint64_t)(uintptr_t)e->rope.p};
  r->timing.host_prep_ms =
      std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t_entry).count();
  run_graphed(r, s, graphable, key, body);
  finish(r, timing, s);
}

// Multi-request batching (SPEC.md:482 continuous
// batching): B independent requests share one fused cache (request b owns rows
// [b*slot, b*slot + T_b)), so one question pass over all B*|Q| rows and one
// sparse pass over all selected rows stream every weight matrix once for the
// whole batch; attention, scoring and top-k run per request on its own cache
// slice (Seg). Each request's result equals its single-request reprocess
// (same kernels, same per-request plans; GEMM rows are independent).
void reprocess_batch(Engine* e, Store* st, const frag_request* reqs, int B, int slot, const frag_reprocess_opts* o,
                     cudaStream_t s, Result* r) {
  std::lock_guard<std::recursive_mutex> gpu_lock(device_mutex(e->device));
  const auto& c = e->cfg;
  if (!r || r->eng != e) fail(FRAG_E_CONTRACT, "result does not belong to this engine");
  if (!st) fail(FRAG_E_CONTRACT, "store is null");
  if (st->device != e->device) fail(FRAG_E_CONTRACT, "store and engine are on different devices");
  if (B < 1 || !reqs) fail(FRAG_E_CONTRACT, "batch needs at least one request");
  if (slot < 1 || (long)B * slot > r->max_tokens)
    fail(FRAG_E_CONTRACT, "batch of " + std::to_string(B) + " x " + std::to_string(slot) +
                              " rows exceeds the result capacity " + std::to_string(r->max_tokens));
  if (o && (o->inject_crit || o->all_logits || o->selector != FRAG_SELECT_QUERY_GUIDED))
    fail(FRAG_E_CONTRACT, "batched reprocess supports the query-guided selector with last-row logits only");
  DeviceGuard dg(e->device);
  const bool timing = o && o->timing;
  const bool raw = o && o->raw_scores;
  PinGuard pins{st, {}};
  std::vector<std::vector<Record*>> recs(B);
  std::vector<SysKV*> skv(B);
  std::vector<Result::BatchReq> br(B);
  int Qtot = 0, Ntot = 0, Mtot = 0, maxN = 0, maxQ = 0;
  e->ensure_rope(slot);
  for (int b = 0; b < B; ++b) {
    const frag_request& q = reqs[b];
    if (q.n_q < 1 || !q.question) fail(FRAG_E_CONTRACT, "every request needs a question");
    if (q.n_sys < 0 || q.n_chunks < 0 || (q.n_sys > 0 && !q.sys) || (q.n_chunks > 0 && !q.chunk_ids))
      fail(FRAG_E_CONTRACT, "bad request");
    if (!(q.recompute_ratio >= 0.f && q.recompute_ratio <= 1.f))
      fail(FRAG_E_CONTRACT, "recompute_ratio must lie in [0, 1]");
    for (int i = 0; i < q.n_q; ++i)
      if (q.question[i] < 0 || q.question[i] >= c.vocab) fail(FRAG_E_CONTRACT, "question token out of vocabulary");
    int N = 0;
    for (int i = 0; i < q.n_chunks; ++i) {
      recs[b].push_back(store_fetch(st, q.chunk_ids[i]));
      pins.ids.push_back(q.chunk_ids[i]);
      N += recs[b].back()->n_tok;
    }
    const int T = q.n_sys + N + q.n_q;
    if (T > slot) fail(FRAG_E_CONTRACT, "request " + std::to_string(b) + " has " + std::to_string(T) +
                                            " tokens, more than the batch slot of " + std::to_string(slot));
    const int k = (int)std::floor((double)q.recompute_ratio * (double)N + 0.5);
    br[b] = {T, q.n_sys, N, q.n_q, k, Mtot, {}};
    skv[b] = get_sys_kv(e, q.sys, q.n_sys, s);
    Qtot += q.n_q;
    Ntot += N;
    Mtot += k + q.n_q;
    maxN = std::max(maxN, N);
    maxQ = std::max(maxQ, q.n_q);
  }
  r->T = B * slot;
  r->S = 0;
  r->N = Ntot;
  r->nq = Qtot;
  r->k_sel = Mtot - Qtot;
  r->M = Mtot;
  r->logit_rows = B;
  r->rows_per_seq = slot;
  r->logits_on_device = o && o->logits_on_device;
  r->batch = br;
  const size_t kvc = (size_t)c.n_kv_heads * c.head_dim;
  // shared V pages: every request reads its chunks' V in place (a record
  // reused by several requests of the batch is one set of pages)
  bool vsh = shared_v_enabled() && fragk::attn_shared_v_supported(c.head_dim);
  for (int b = 0; b < B && vsh; ++b)
    vsh = br[b].N > 0 && 2L * br[b].k <= br[b].N && fragk::vpatch_plan_fits(slot, (int)recs[b].size() + 1) &&
          records_local(e, recs[b]);
  if (vsh) {
    if (!r->vshared) r->v_fused.release();
    r->vshared = true;
    r->v_materialized = false;
    r->v_tail_row0 = 0x7fffffff;  // every fresh row at its GEMM row's slot
    r->v_tail_slot0 = 0;
  } else {
    use_private_v(r);
  }

  // ---- host prep
  r->staging.ensure(64 * 1024 + (size_t)(pins.ids.size() + 2 * B) * (64 + c.head_dim * 4 + sizeof(fragk::VSeg)) +
                    (size_t)B * 2 * sizeof(fragk::VPlanArgs) + (size_t)(4 * Qtot + 4 * B) * 4);
  Stage stg(r->staging);
  std::vector<StitchPart> parts;
  for (int b = 0; b < B; ++b) parts.push_back(StitchPart{skv[b], &recs[b], br[b].S, b * slot});
  StitchPlan sp = stitch_prepare_parts(e, r, s, stg, parts);
  std::vector<int> cofs(B), qofs(B);
  {
    int co = 0, qo = 0;
    int* qh = stg.take<int>(Qtot);
    int* rows_h = stg.take<int>(Qtot);
    for (int b = 0; b < B; ++b) {
      cofs[b] = co;
      qofs[b] = qo;
      for (Record* rec : recs[b]) {
        check_cuda(cudaMemcpyAsync(r->chunk_tok.as<int>() + co, rec->tok.p, rec->n_tok * sizeof(int),
                                   cudaMemcpyDeviceToDevice, s),
                   "chunk tokens");
        co += rec->n_tok;
      }
      for (int i = 0; i < br[b].nq; ++i) {
        qh[qo + i] = reqs[b].question[i];
        rows_h[qo + i] = b * slot + br[b].T - br[b].nq + i;
      }
      qo += br[b].nq;
    }
    check_cuda(cudaMemcpyAsync(r->q_tok.p, qh, Qtot * sizeof(int), cudaMemcpyHostToDevice, s), "q tok");
    check_cuda(cudaMemcpyAsync(r->plan_rows.p, rows_h, Qtot * sizeof(int), cudaMemcpyHostToDevice, s), "q rows");
    check_cuda(cudaMemcpyAsync(r->plan_tok.p, r->q_tok.p, Qtot * sizeof(int), cudaMemcpyDeviceToDevice, s), "q plan");
    int* map_h = stg.take<int>(B);
    // logits rows: the sparse pass keeps each request's last row, compacted
    // after the plan rows (last-layer pruning of run_rows)
    const bool compact = Mtot + B <= r->max_tokens;
    for (int b = 0; b < B; ++b) map_h[b] = compact ? Mtot + b : br[b].plan_off + br[b].k + br[b].nq - 1;
    check_cuda(cudaMemcpyAsync(r->row_map.p, map_h, B * sizeof(int), cudaMemcpyHostToDevice, s), "map");
  }
  if (vsh) {
    std::vector<VPart> vp;
    for (int b = 0; b < B; ++b)
      vp.push_back(VPart{skv[b], &recs[b], br[b].S, b * slot, br[b].T, br[b].nq, br[b].k, br[b].plan_off, qofs[b],
                         br[b].plan_off + br[b].k});
    vshared_prepare(e, r, s, stg, vp, slot, Mtot);
  }
  if (maxN > 0) {
    r->part_ms.ensure((size_t)((maxN + 31) / 32) * maxQ * c.n_heads * sizeof(float2));
    r->row_ms.ensure((size_t)maxQ * c.n_heads * sizeof(float2));
    r->score_col.ensure(fragk::score_col_part_elems(maxQ, c.n_heads, c.n_kv_heads, maxN) * sizeof(float));
    r->score_q.ensure(fragk::score_q_split_elems(maxQ, c.n_heads, c.n_kv_heads, c.head_dim) * sizeof(bf16));
  }
  r->lm_x.ensure((size_t)B * c.d_model * sizeof(bf16));
  r->logits.ensure((size_t)B * c.vocab * sizeof(float));
  if (!r->logits_on_device) r->logits_host.ensure((size_t)B * c.vocab * sizeof(float));
  std::vector<Seg> qsegs, psegs;
  for (int b = 0; b < B; ++b) {
    qsegs.push_back(Seg{qofs[b], br[b].nq, b * slot, br[b].T, b});
    psegs.push_back(Seg{br[b].plan_off, br[b].k + br[b].nq, b * slot, br[b].T, b});
  }

  // ---- device body: captured into a CUDA graph per batch shape (like a
  // single request's body) and replayed from the third batch of that shape on
  auto body = [&](cudaStream_t s) {
    ev_record(r, timing, 0, s);
    stitch_launch(e, r, s, sp);
    ev_record(r, timing, 1, s);
    vplan_launch(e, r, s, 0);
    run_rows(e, r, s, Qtot, slot, PASS_QUESTION, nullptr, 0, 0, nullptr, &qsegs);
    ev_record(r, timing, 2, s);
    for (int b = 0; b < B; ++b) {
      const auto& q = br[b];
      if (q.N > 0) {
        fragk::ScoreArgs a{};
        a.q = r->q_final.as<float>() + (size_t)qofs[b] * c.n_heads * c.head_dim;
        a.k = r->k_fused.as<bf16>() + (size_t)(c.layers - 1) * r->max_tokens * kvc + (size_t)b * slot * kvc;
        a.nq = q.nq;
        a.Hq = c.n_heads;
        a.Hkv = c.n_kv_heads;
        a.dh = c.head_dim;
        a.key_row0 = q.S;
        a.n_keys = q.N;
        a.scale = 1.0f / std::sqrt((float)c.head_dim);
        a.part_ms = r->part_ms.as<float2>();
        a.row_ms = r->row_ms.as<float2>();
        a.scores = r->scores.as<float>() + cofs[b];
        a.raw = raw;
        a.col_part = r->score_col.as<float>();
        a.q_split = r->score_q.as<bf16>();
        Scoped sc(e->prof, s, KC_SELECT, 4.0 * q.nq * c.n_heads * (double)q.N * c.head_dim,
                  2.0 * q.N * (double)kvc * 2);
        sc.launched(fragk::qg_score(a, s));
      }
      Scoped sc(e->prof, s, KC_SELECT, 0, 4.0 * q.N * 6);
      sc.launched(fragk::topk_plan(r->scores.as<float>() + cofs[b], q.N, q.k, b * slot + q.S,
                                   r->chunk_tok.as<int>() + cofs[b], r->q_tok.as<int>() + qofs[b], q.nq,
                                   b * slot + q.T - q.nq, r->plan_rows.as<int>() + q.plan_off,
                                   r->plan_tok.as<int>() + q.plan_off, s));
    }
    peek("batch select");
    vplan_launch(e, r, s, 1);
    ev_record(r, timing, 3, s);
    run_rows(e, r, s, Mtot, slot, PASS_FULL, nullptr, 0, 0, nullptr, &psegs, -1);
    ev_record(r, timing, 4, s);
    {
      const int d = c.d_model;
      {
        Scoped sc(e->prof, s, KC_NORM, 0, (double)B * d * 6);
        fragk::rmsnorm(r->h.as<float>(), B, d, e->final_norm, c.norm_eps, r->lm_x.as<bf16>(), s, r->row_map.as<int>());
        sc.launched(1);
      }
      fragk::EpiParams ep;
      ep.ws = r->gemm_ws.as<float>();
      ep.ws_bytes = r->gemm_ws.bytes;
      ep.counters = r->gemm_cnt.as<int>();
      ep.counters_cap = gemm_counter_cap(r);
      ep.out_f32 = r->logits.as<float>();
      ep.ldo = c.vocab;
      Scoped sc(e->prof, s, gemm_class(B), 2.0 * B * (double)c.vocab * d, 2.0 * c.vocab * (double)d);
      sc.launched(fragk::gemm_bf16_tc(r->lm_x.as<bf16>(), e->lm_head, B, c.vocab, d, fragk::EPI_STORE_F32, ep, s));
    }
    peek("batch lm_head");
    ev_record(r, timing, 5, s);
    logits_d2h(r, s);
  };
  GraphKey key{B * slot, -2 - B, Ntot, Qtot, Mtot - Qtot, 0, 0, (int)raw, (int)r->logits_on_device, sp.n_desc,
               sp.max_rows, vsh ? 4000 : 0, (uint64_t)(uintptr_t)e->rope.p};
  for (const auto& q : br)  // batch shape: every request's exact (T, S, N, |Q|, k)
    key.shapes.insert(key.shapes.end(), {q.T, q.S, q.N, q.nq, q.k});
  run_graphed(r, s, !timing && !e->prof.on, key, body);
  // per-request critical positions (host copies for frag_result_batch_crit)
  std::vector<int32_t> plan_h((size_t)Mtot);
  check_cuda(cudaMemcpyAsync(plan_h.data(), r->plan_rows.p, Mtot * sizeof(int), cudaMemcpyDeviceToHost, s), "plan");
  finish(r, timing, s);
  for (int b = 0; b < B; ++b) {
    r->batch[b].crit.resize(br[b].k);
    for (int i = 0; i < br[b].k; ++i) r->batch[b].crit[i] = plan_h[br[b].plan_off + i] - b * slot + 1;
  }
}

void full_prefill(Engine* e, const int32_t* sys, int n_sys, const int32_t* tokens, int n_tok,
                  const frag_reprocess_opts* o, cudaStream_t s, Result* r) {
  std::lock_guard<std::recursive_mutex> gpu_lock(device_mutex(e->device));
  const auto& c = e->cfg;
  if (!r || r->eng != e) fail(FRAG_E_CONTRACT, "result does not belong to this engine");
  if (n_tok < 1) fail(FRAG_E_CONTRACT, "full prefill needs at least one token");
  for (int i = 0; i < n_tok; ++i)
    if (tokens[i] < 0 || tokens[i] >= c.vocab) fail(FRAG_E_CONTRACT, "token out of vocabulary");
  DeviceGuard dg(e->device);
  const bool timing = o && o->timing;
  const int S = n_sys, T = S + n_tok;
  if (T > r->max_tokens) fail(FRAG_E_CONTRACT, "prompt exceeds the result capacity");
  use_private_v(r);  // every row is fresh
  e->ensure_rope(T);
  SysKV* skv = get_sys_kv(e, sys, n_sys, s);
  r->T = T;
  r->rows_per_seq = 0;
  r->batch.clear();
  r->S = S;
  r->N = n_tok;
  r->nq = 0;
  r->k_sel = n_tok;
  r->M = n_tok;
  r->logit_rows = 1;
  r->staging.ensure(64 * 1024 + (size_t)8 * T + 1024);
  Stage stg(r->staging);
  ev_record(r, timing, 0, s);
  stitch(e, r, s, stg, skv, {}, S);
  ev_record(r, timing, 1, s);
  ev_record(r, timing, 2, s);
  int* rows_h = stg.take<int>(n_tok);
  int* tok_h = stg.take<int>(n_tok);
  for (int i = 0; i < n_tok; ++i) rows_h[i] = S + i, tok_h[i] = tokens[i];
  check_cuda(cudaMemcpyAsync(r->plan_rows.p, rows_h, n_tok * sizeof(int), cudaMemcpyHostToDevice, s), "rows");
  check_cuda(cudaMemcpyAsync(r->plan_tok.p, tok_h, n_tok * sizeof(int), cudaMemcpyHostToDevice, s), "tok");
  int* map_h = stg.take<int>(1);
  map_h[0] = n_tok - 1;
  check_cuda(cudaMemcpyAsync(r->row_map.p, map_h, sizeof(int), cudaMemcpyHostToDevice, s), "map");
  ev_record(r, timing, 3, s);
  run_rows(e, r, s, n_tok, T, PASS_FULL, r->row_map.as<int>(), 1, 0, nullptr, nullptr, 1);
  ev_record(r, timing, 4, s);
  ev_record(r, timing, 5, s);
  r->logits_on_device = o && o->logits_on_device;
  if (!r->logits_on_device) r->logits_host.ensure((size_t)c.vocab * sizeof(float));
  logits_d2h(r, s);
  finish(r, timing, s);
}

void kv_deviation(Engine* e, Store* st, const int32_t* sys, int n_sys, const frag_chunk_id* ids, int n_chunks,
                  int n_layers, cudaStream_t s, Result* r, float* dev_host) {
  std::lock_guard<std::recursive_mutex> gpu_lock(device_mutex(e->device));
  const auto& c = e->cfg;
  if (!r || r->eng != e) fail(FRAG_E_CONTRACT, "result does not belong to this engine");
  if (!st) fail(FRAG_E_CONTRACT, "store is null");
  if (st->device != e->device) fail(FRAG_E_CONTRACT, "store and engine are on different devices");
  if (n_layers < 1 || n_layers > c.layers) fail(FRAG_E_CONTRACT, "n_layers must lie in [1, layers]");
  if (n_sys < 0 || n_chunks < 1 || !ids) fail(FRAG_E_CONTRACT, "kv_deviation needs at least one chunk");
  DeviceGuard dg(e->device);
  PinGuard pins{st, {}};
  std::vector<Record*> recs;
  for (int i = 0; i < n_chunks; ++i) {
    recs.push_back(store_fetch(st, ids[i]));
    pins.ids.push_back(ids[i]);
  }
  const int S = n_sys;
  int N = 0;
  for (Record* rec : recs) N += rec->n_tok;
  const int T = S + N;
  if (T > r->max_tokens) fail(FRAG_E_CONTRACT, "context exceeds the result capacity");
  use_private_v(r);  // the Full-Attention pass rewrites every chunk row
  e->ensure_rope(T);
  SysKV* skv = get_sys_kv(e, sys, n_sys, s);
  r->T = T;
  r->rows_per_seq = 0;
  r->batch.clear();
  r->S = S;
  r->N = N;
  r->nq = 0;
  r->k_sel = 0;
  r->M = 0;
  r->logit_rows = 0;
  const size_t kvc = (size_t)c.n_kv_heads * c.head_dim;
  r->fr_save.ensure((size_t)2 * n_layers * N * kvc * sizeof(bf16));
  r->dev.ensure((size_t)N * n_layers * 2 * sizeof(float));
  r->staging.ensure(64 * 1024 + (size_t)(n_chunks + 2) * (64 + c.head_dim * 4) + (size_t)8 * N);
  Stage stg(r->staging);
  stitch(e, r, s, stg, skv, recs, S);
  int* rows_h = stg.take<int>(N);
  for (int i = 0; i < N; ++i) rows_h[i] = S + i;
  check_cuda(cudaMemcpyAsync(r->plan_rows.p, rows_h, N * sizeof(int), cudaMemcpyHostToDevice, s), "fa rows");
  int off = 0;
  for (Record* rec : recs) {
    check_cuda(cudaMemcpyAsync(r->plan_tok.as<int>() + off, rec->tok.p, rec->n_tok * sizeof(int),
                               cudaMemcpyDeviceToDevice, s),
               "fa tokens");
    off += rec->n_tok;
  }
  deviation_body(e, r, s, S, N, n_layers, r->dev.as<float>(), nullptr, 0);
  check_cuda(cudaMemcpyAsync(dev_host, r->dev.p, (size_t)N * n_layers * 2 * sizeof(float), cudaMemcpyDefault, s),
             "deviation D2H");
  sync_checked(e, r, s, "kv_deviation");
}

void decode(Engine* e, Result* r, int n_new, cudaStream_t s, int32_t* out_host) {
  std::lock_guard<std::recursive_mutex> gpu_lock(device_mutex(e->device));
  const auto& c = e->cfg;
  if (!r || r->eng != e) fail(FRAG_E_CONTRACT, "result does not belong to this engine");
  if (n_new < 1) fail(FRAG_E_CONTRACT, "max_new_tokens must be >= 1");
  if (!out_host) fail(FRAG_E_CONTRACT, "tokens_out is null");
  if (r->T <= 0 || r->logit_rows < 1) fail(FRAG_E_CONTRACT, "decode needs a preceding reprocess or full prefill");
  if (r->rows_per_seq > 0) fail(FRAG_E_CONTRACT, "decode after a batched reprocess is not supported");
  const int T0 = r->T;
  if (T0 + n_new - 1 > r->max_tokens)
    fail(FRAG_E_CONTRACT, "decoded tokens exceed the result capacity (" + std::to_string(r->max_tokens) + ")");
  DeviceGuard dg(e->device);
  // every step attends over the result's whole capacity (keys past the row's
  // position are masked by position, split-KV ranges past it are empty), so a
  // step's launches do not depend on its position and replay from one graph
  const int T_cap = r->max_tokens;
  e->ensure_rope(T_cap);
  r->dec_tok.ensure((size_t)(n_new + 1) * sizeof(int));
  r->staging.ensure((size_t)n_new * sizeof(int) + 64);
  int* stage = r->staging.as<int>();
  stage[0] = 0;  // the single decode row is logits row 0
  stage[1] = 0;  // token slot counter
  int* cnt = r->dec_tok.as<int>();  // [0] slot counter, [1..] tokens (fixed addresses for the graph)
  int* toks = cnt + 1;
  check_cuda(cudaMemcpyAsync(r->row_map.p, stage, sizeof(int), cudaMemcpyHostToDevice, s), "row map");
  check_cuda(cudaMemcpyAsync(cnt, stage + 1, sizeof(int), cudaMemcpyHostToDevice, s), "slot counter");
  auto argmax = [&](const float* logits, int next_row, cudaStream_t bs) {
    Scoped sc(e->prof, bs, KC_SELECT, 0, 4.0 * c.vocab);
    sc.launched(fragk::greedy_argmax(logits, c.vocab, toks, cnt, r->plan_tok.as<int>(),
                                     r->plan_rows.as<int>(), next_row, bs));
  };
  // token 0 = argmax of the prefill's last logits row; its row is T0 (0-based)
  argmax(r->logits.as<float>() + (size_t)(r->logit_rows - 1) * c.vocab, T0, s);
  // step: one row through every layer at plan_rows[0], logits row 0, argmax ->
  // next token and plan_rows[0] + 1 (graph-replayed after the first step)
  auto step = [&](cudaStream_t bs) {
    run_rows(e, r, bs, 1, T_cap, PASS_FULL, r->row_map.as<int>(), 1);
    argmax(r->logits.as<float>(), -1, bs);
  };
  const bool graphable = !e->prof.on;
  GraphKey key{T_cap, -1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, (uint64_t)(uintptr_t)e->rope.p};
  for (int i = 1; i < n_new; ++i) run_graphed(r, s, graphable, key, step);
  peek("decode");
  check_cuda(cudaMemcpyAsync(stage, toks, (size_t)n_new * sizeof(int), cudaMemcpyDeviceToHost, s), "tokens");
  if (n_new > 1) {
    r->logit_rows = 1;
    if (!r->logits_on_device) {
      r->logits_host.ensure((size_t)c.vocab * sizeof(float));
      logits_d2h(r, s);
    }
  }
  r->last_stream = s;
  sync_checked(e, r, s, "decode");
  std::memcpy(out_host, stage, (size_t)n_new * sizeof(int));
  r->T = T0 + n_new - 1;  // the fused cache now also holds the decoded tokens' K/V
  if (r->vshared && !r->vseq.empty()) r->vseq[0].T = r->T;
  r->v_materialized = false;
  r->timing_valid = false;
}

void preprocess_isolated(Engine* e, Store* st, const int32_t* sys, int n_sys, const int32_t* tokens, int n_tok,
                         bool overwrite, frag_chunk_id* id_out) {
  std::lock_guard<std::recursive_mutex> gpu_lock(device_mutex(e->device));
  const auto& c = e->cfg;
  if (n_tok < 1) fail(FRAG_E_CONTRACT, "chunk must have at least one token (SPEC.md:197)");
  for (int i = 0; i < n_tok; ++i)
    if (tokens[i] < 0 || tokens[i] >= c.vocab) fail(FRAG_E_CONTRACT, "token out of vocabulary");
  if (st->device != e->device) fail(FRAG_E_CONTRACT, "store and engine are on different devices");
  frag_chunk_id id;
  hash_tokens(tokens, n_tok, 0, &id);
  {
    std::shared_lock<std::shared_mutex> g(st->mu);
    if (!overwrite && st->recs.count(key_of(id)))
      fail(FRAG_E_STORE, "duplicate chunk record without overwrite (SPEC.md:269)");
  }
  DeviceGuard dg(e->device);
  cudaStream_t s;
  check_cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  struct SG {
    cudaStream_t s;
    ~SG() { cudaStreamDestroy(s); }
  } sg{s};
  const int S = n_sys, T = S + n_tok;
  e->ensure_rope(T);
  SysKV* skv = get_sys_kv(e, sys, n_sys, s);
  std::lock_guard<std::mutex> g(e->mu);  // scratch result is shared
  Result* r = scratch_for(e, T);
  r->staging.ensure(64 * 1024 + (size_t)8 * T + 1024);
  Stage stg(r->staging);
  stitch(e, r, s, stg, skv, {}, S);
  int* rows_h = stg.take<int>(n_tok);
  int* tok_h = stg.take<int>(n_tok);
  for (int i = 0; i < n_tok; ++i) rows_h[i] = S + i, tok_h[i] = tokens[i];
  check_cuda(cudaMemcpyAsync(r->plan_rows.p, rows_h, n_tok * sizeof(int), cudaMemcpyHostToDevice, s), "rows");
  check_cuda(cudaMemcpyAsync(r->plan_tok.p, tok_h, n_tok * sizeof(int), cudaMemcpyHostToDevice, s), "tok");
  run_rows(e, r, s, n_tok, T, PASS_KV_ONLY, nullptr, 0);
  sync_checked(e, r, s, "preprocess");  // never store a record computed by a faulted grid
  const size_t kvc = (size_t)c.n_kv_heads * c.head_dim;
  store_put(st, id, tokens, n_tok, S + 1, FRAG_VARIANT_ISOLATED, r->k_fused.as<bf16>() + (size_t)S * kvc,
            r->v_fused.as<bf16>() + (size_t)S * kvc, overwrite, (size_t)r->max_tokens * kvc, s);
  check_cuda(cudaStreamSynchronize(s), "preprocess");
  // cached under context (S, [chunk]) (alternative_path_match index)
  frag_chunk_id sid;
  if (n_sys > 0) hash_tokens(sys, n_sys, 0, &sid);
  store_register_prefix(st, n_sys > 0 ? &sid : nullptr, &id, 1);
  if (id_out) *id_out = id;
}

// preprocess_fused (Eq. 10): C_i prefilled
// against cat(KV_S, its top-n neighbours' ISOLATED records stitched exactly as
// the online Full Reuse path) at positions [|X|+1 : |X|+|C_i|], X = S + the
// neighbours. Neighbours in the given order (descending similarity), truncated
// from the tail to the fused-context budget; the record (variant FUSED,
// native_start |X|+1) goes to dst. With no neighbours the K/V are exactly
// preprocess_isolated's (same launches, bit-identical record data).
void preprocess_fused(Engine* e, Store* src, Store* dst, const int32_t* sys, int n_sys, const int32_t* tokens,
                      int n_tok, const frag_chunk_id* nb, int n_nb, int budget, bool overwrite, frag_chunk_id* id_out) {
  std::lock_guard<std::recursive_mutex> gpu_lock(device_mutex(e->device));
  const auto& c = e->cfg;
  if (n_tok < 1) fail(FRAG_E_CONTRACT, "chunk must have at least one token (SPEC.md:197)");
  if (n_nb < 0 || (n_nb > 0 && !nb)) fail(FRAG_E_CONTRACT, "bad neighbour list");
  for (int i = 0; i < n_tok; ++i)
    if (tokens[i] < 0 || tokens[i] >= c.vocab) fail(FRAG_E_CONTRACT, "token out of vocabulary");
  if (src->device != e->device || dst->device != e->device)
    fail(FRAG_E_CONTRACT, "stores and engine are on different devices");
  if (budget <= 0) budget = 2048;  // SPEC.md design decision: default fused-context budget
  frag_chunk_id id;
  hash_tokens(tokens, n_tok, 0, &id);
  {
    std::shared_lock<std::shared_mutex> g(dst->mu);
    if (!overwrite && dst->recs.count(key_of(id)))
      fail(FRAG_E_STORE, "duplicate chunk record without overwrite (SPEC.md:269)");
  }
  PinGuard pins{src, {}};
  std::vector<Record*> recs;
  int X = n_sys;
  for (int i = 0; i < n_nb; ++i) {
    Record* rec = nullptr;
    try {
      rec = store_fetch(src, nb[i]);
    } catch (const Error&) {
      static const char* hx = "0123456789abcdef";
      std::string h;
      for (int b = 0; b < 16; ++b) h += hx[nb[i].bytes[b] >> 4], h += hx[nb[i].bytes[b] & 15];
      fail(FRAG_E_STORE, "missing neighbour record " + h + " (SPEC.md:357)");
    }
    pins.ids.push_back(nb[i]);
    if (rec->variant != FRAG_VARIANT_ISOLATED)
      fail(FRAG_E_CONTRACT, "Eq. 10 neighbours must be ISOLATED records (two-round fusion is out of scope)");
    if (X - n_sys + rec->n_tok > budget) break;  // truncate from the tail of the list
    recs.push_back(rec);
    X += rec->n_tok;
  }
  DeviceGuard dg(e->device);
  cudaStream_t s;
  check_cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  struct SG {
    cudaStream_t s;
    ~SG() { cudaStreamDestroy(s); }
  } sg{s};
  const int T = X + n_tok;
  e->ensure_rope(T);
  SysKV* skv = get_sys_kv(e, sys, n_sys, s);
  std::lock_guard<std::mutex> g(e->mu);  // scratch result is shared
  Result* r = scratch_for(e, T);
  r->staging.ensure(64 * 1024 + (size_t)(recs.size() + 2) * (64 + c.head_dim * 4) + (size_t)8 * T + 1024);
  Stage stg(r->staging);
  stitch(e, r, s, stg, skv, recs, n_sys);  // KV_S + neighbours at consecutive positions (Full Reuse)
  int* rows_h = stg.take<int>(n_tok);
  int* tok_h = stg.take<int>(n_tok);
  for (int i = 0; i < n_tok; ++i) rows_h[i] = X + i, tok_h[i] = tokens[i];
  check_cuda(cudaMemcpyAsync(r->plan_rows.p, rows_h, n_tok * sizeof(int), cudaMemcpyHostToDevice, s), "rows");
  check_cuda(cudaMemcpyAsync(r->plan_tok.p, tok_h, n_tok * sizeof(int), cudaMemcpyHostToDevice, s), "tok");
  run_rows(e, r, s, n_tok, T, PASS_KV_ONLY, nullptr, 0);
  sync_checked(e, r, s, "preprocess_fused");
  const size_t kvc = (size_t)c.n_kv_heads * c.head_dim;
  store_put(dst, id, tokens, n_tok, X + 1, FRAG_VARIANT_FUSED,
            r->k_fused.as<bf16>() + (size_t)X * kvc, r->v_fused.as<bf16>() + (size_t)X * kvc, overwrite,
            (size_t)r->max_tokens * kvc, s);
  check_cuda(cudaStreamSynchronize(s), "preprocess_fused");
  {  // cached under context (S, [neighbours used..., chunk])
    std::vector<frag_chunk_id> path;
    for (Record* rec : recs) path.push_back(rec->id);
    path.push_back(id);
    frag_chunk_id sid;
    if (n_sys > 0) hash_tokens(sys, n_sys, 0, &sid);
    store_register_prefix(dst, n_sys > 0 ? &sid : nullptr, path.data(), (int)path.size());
  }
  if (id_out) *id_out = id;
}

}  // namespace fragimpl

// Tooling (tools/r0_check.py; not part of the frag C API): the allocation
// epoch that invalidates captured request graphs.
extern "C" __attribute__((visibility("default"))) unsigned long long frag_debug_alloc_epoch() {
  return (unsigned long long)fragimpl::g_alloc_epoch.load();
}
