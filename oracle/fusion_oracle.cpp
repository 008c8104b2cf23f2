// ============================================================================
// CPU ORACLE — test infrastructure only. NOT part of the product path.
//
// A fp32 C++ restatement of the reference's online reprocessing stage, written
// from /root/reference/SPEC.md (the reference ships no implementation, see
// SURVEY.md §0) and PAPER.md. Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load it, and only as the
// checker or the timed CPU baseline. libfrag.so never links or calls it.
//
// Parity pinning: the Rng restatement is pinned bit-exactly
// to the reference's own header (common.hpp:45-100) through golden vectors
// produced by oracle/_ref/rng_kat (compiled from /root/reference by
// oracle/Makefile). The model / stitch / select / sparse-prefill arithmetic has
// no reference implementation to run; it is pinned only by the SPEC.md worked
// examples and property oracles (tests/test_oracle_spec.py): "parity partially
// pinned".
//
// Cited reference lines:
//   Rng                  common.hpp:45-100
//   apply_rope/shift     SPEC.md:22-49, PAPER.md:1013-1049 (Appendix A)
//   forward              SPEC.md:103-111 (pre-norm, RMS, gated FFN, scale 1/sqrt(dh))
//   last_layer_query_states SPEC.md:112-120
//   q_sparse_attn        SPEC.md:153-161; build_equivalent_mask SPEC.md:162-170
//   stitch_full_reuse    SPEC.md:399-407 (Eq. 6)
//   select_query_guided
//   kv_deviation         SPEC.md:408-416 (Eq. 7)
//   select_cacheblend    SPEC.md:417-425 (Eq. 8)
//   sparse_prefill       SPEC.md:435-444 (Eq. 9)
//   preprocess_isolated  SPEC.md:344-352 (Eq. 5)
// ============================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

extern "C" {

typedef struct {
  int32_t layers, d_model, n_heads, n_kv_heads, head_dim, ffn_dim, vocab;
  double rope_base;
  float norm_eps;
} orc_cfg;

}  // extern "C"

namespace {

// ------------------------------------------------------------------ Rng (common.hpp:45-100)
struct Rng {
  uint64_t state;
  bool has_spare = false;
  double spare = 0.0;
  explicit Rng(uint64_t s) : state(s) {}
  uint64_t next_u64() {
    uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  uint32_t next_u32() { return (uint32_t)(next_u64() >> 32); }
  double next_double() { return (double)(next_u64() >> 11) * 0x1.0p-53; }
  float next_float() { return (float)next_double(); }
  uint64_t below(uint64_t n) {
    uint64_t threshold = (0 - n) % n;
    for (;;) {
      uint64_t r = next_u64();
      if (r >= threshold) return r % n;
    }
  }
  double normal() {
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    double u1 = 0.0;
    do {
      u1 = next_double();
    } while (u1 <= 0.0);
    double u2 = next_double();
    double mag = std::sqrt(-2.0 * std::log(u1));
    spare = mag * std::sin(6.283185307179586477 * u2);
    has_spare = true;
    return mag * std::cos(6.283185307179586477 * u2);
  }
  float normal_f(float sigma) { return (float)normal() * sigma; }
};

uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
uint64_t splitmix_at(uint64_t seed, uint64_t n) { return mix64(seed + (n + 1) * 0x9e3779b97f4a7c15ULL); }

inline float bf16r(float f) {  // round-to-nearest-even to bfloat16, returned as float
  uint32_t b;
  std::memcpy(&b, &f, 4);
  if ((b & 0x7f800000u) == 0x7f800000u) return f;
  b += 0x7fffu + ((b >> 16) & 1u);
  b &= 0xffff0000u;
  float o;
  std::memcpy(&o, &b, 4);
  return o;
}

// ------------------------------------------------------------------ model
struct Layer {
  std::vector<float> wq, wk, wv, wo, wg, wu, wd, attn_norm, ffn_norm;
};
struct Model {
  orc_cfg c;
  std::vector<float> emb, lm_head, final_norm;
  std::vector<Layer> layers;
  std::vector<double> theta;  // theta_i = base^(-2i/d), i = 1..d/2
};

// C[M,N] = A[M,K] . W[N,K]^T (+ C if accumulate). Register-blocked 2x4 dot
// products with OpenMP over W row blocks; fp32 accumulation per output in a
// fixed order (deterministic for a fixed thread count-independent schedule).
void gemm_nt(const float* A, const float* W, float* Cm, int M, int N, int K, bool accumulate) {
  constexpr int NB = 64;
  const int nblocks = (N + NB - 1) / NB;
#pragma omp parallel for schedule(dynamic, 1) collapse(2)
  for (int nb = 0; nb < nblocks; ++nb) {
    for (int mb = 0; mb < (M + 63) / 64; ++mb) {
      const int n0 = nb * NB, n1 = std::min(N, n0 + NB);
      const int m0 = mb * 64, m1 = std::min(M, m0 + 64);
      for (int i = m0; i < m1; i += 2) {
        const int i2 = std::min(i + 1, m1 - 1);
        const float* a0 = A + (size_t)i * K;
        const float* a1 = A + (size_t)i2 * K;
        for (int j = n0; j < n1; j += 4) {
          const float* w[4];
          for (int t = 0; t < 4; ++t) w[t] = W + (size_t)std::min(j + t, n1 - 1) * K;
          float s[2][4] = {};
          for (int t = 0; t < 4; ++t) {
            float acc0 = 0.f, acc1 = 0.f;
            const float* wt = w[t];
#pragma omp simd reduction(+ : acc0, acc1)
            for (int k = 0; k < K; ++k) {
              acc0 += a0[k] * wt[k];
              acc1 += a1[k] * wt[k];
            }
            s[0][t] = acc0;
            s[1][t] = acc1;
          }
          for (int t = 0; t < 4 && j + t < n1; ++t) {
            float* c0 = Cm + (size_t)i * N + j + t;
            *c0 = accumulate ? *c0 + s[0][t] : s[0][t];
            if (i + 1 < m1) {
              float* c1 = Cm + (size_t)(i + 1) * N + j + t;
              *c1 = accumulate ? *c1 + s[1][t] : s[1][t];
            }
          }
        }
      }
    }
  }
}

void rmsnorm_rows(const float* h, const float* g, float* x, int M, int d, float eps, bool emu) {
#pragma omp parallel for schedule(static)
  for (int i = 0; i < M; ++i) {
    const float* hr = h + (size_t)i * d;
    double ss = 0.0;
    for (int k = 0; k < d; ++k) ss += (double)hr[k] * hr[k];
    const float rs = 1.0f / std::sqrt((float)(ss / d) + eps);
    float* xr = x + (size_t)i * d;
    for (int k = 0; k < d; ++k) {
      const float v = hr[k] * rs * g[k];
      xr[k] = emu ? bf16r(v) : v;
    }
  }
}

// RoPE(k, s) = k cos(s theta) + rotate(k) sin(s theta), rotate(k) = [-k2, k1, -k4, k3, ...]
// (Eq. 20-22). Angles in fp64, cos/sin cast to fp32,
// then one fused multiply-add per output (the same op order as the GPU epilogue and K1).
inline void rope_rotate_pair(float k0, float k1, float c, float s, float& o0, float& o1) {
  o0 = std::fma(k0, c, -(k1 * s));
  o1 = std::fma(k1, c, k0 * s);
}
void rope_apply(float* v, int dh, double pos, const std::vector<double>& theta) {
  for (int i = 0; i < dh / 2; ++i) {
    const double a = pos * theta[i];
    const float c = (float)std::cos(a), s = (float)std::sin(a);
    float o0, o1;
    rope_rotate_pair(v[2 * i], v[2 * i + 1], c, s, o0, o1);
    v[2 * i] = o0;
    v[2 * i + 1] = o1;
  }
}

float silu(float g) { return g / (1.0f + std::exp(-g)); }

struct Cache {
  int cap = 0;
  float* k = nullptr;    // [L][cap][Hkv][dh]
  float* v = nullptr;
  int32_t* pos = nullptr;  // [cap] 1-based position held by each row, 0 = empty
};

// Generic position-keyed forward: new rows (tokens, 1-based
// positions, cache slots) against the cache; fresh K/V of every new row are
// scattered into its slot before that layer's attention, so earlier fresh rows
// are visible in the same pass. Visibility: mask[i][j] if given,
// else cache row j valid and pos[j] <= positions[i].
// stop_layer_q: if >= 0, return after the QKV projection of the final layer with
// post-RoPE queries in q_out (last_layer_query_states).
// n_layers > 0 runs only the first n_layers layers (with stop_after_last_q the
// pass ends after layer n_layers-1's QKV: kv_deviation's FA pass).
void forward(const Model& m, int n, const int32_t* tokens, const int32_t* positions, const int32_t* slots,
             Cache& cache, const uint8_t* mask, float* logits, int n_logit_rows, const int32_t* logit_rows,
             float* q_out, bool stop_after_last_q, bool emu, int n_layers = 0) {
  const auto& c = m.c;
  const int L = (n_layers > 0 && n_layers < c.layers) ? n_layers : c.layers;
  const int d = c.d_model, Hq = c.n_heads, Hkv = c.n_kv_heads, dh = c.head_dim, F = c.ffn_dim;
  const int qc = Hq * dh, kc = Hkv * dh, G = Hq / Hkv;
  const float scale = 1.0f / std::sqrt((float)dh);
  std::vector<float> h((size_t)n * d), x((size_t)n * d), q((size_t)n * qc), kk((size_t)n * kc),
      vv((size_t)n * kc), o((size_t)n * qc), gg((size_t)n * F), uu((size_t)n * F);
  for (int i = 0; i < n; ++i)
    std::memcpy(&h[(size_t)i * d], &m.emb[(size_t)tokens[i] * d], d * sizeof(float));
  for (int i = 0; i < n; ++i) cache.pos[slots[i]] = positions[i];
  for (int l = 0; l < L; ++l) {
    const Layer& W = m.layers[l];
    rmsnorm_rows(h.data(), W.attn_norm.data(), x.data(), n, d, c.norm_eps, emu);
    gemm_nt(x.data(), W.wq.data(), q.data(), n, qc, d, false);
    gemm_nt(x.data(), W.wk.data(), kk.data(), n, kc, d, false);
    gemm_nt(x.data(), W.wv.data(), vv.data(), n, kc, d, false);
    const bool last_q = stop_after_last_q && l == L - 1;
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) {
      for (int hh = 0; hh < Hq; ++hh) rope_apply(&q[(size_t)i * qc + hh * dh], dh, positions[i], m.theta);
      for (int hh = 0; hh < Hkv; ++hh) rope_apply(&kk[(size_t)i * kc + hh * dh], dh, positions[i], m.theta);
      if (last_q && q_out) std::memcpy(q_out + (size_t)i * qc, &q[(size_t)i * qc], qc * sizeof(float));
      float* ck = cache.k + ((size_t)l * cache.cap + slots[i]) * kc;
      float* cv = cache.v + ((size_t)l * cache.cap + slots[i]) * kc;
      for (int t = 0; t < kc; ++t) {
        ck[t] = emu ? bf16r(kk[(size_t)i * kc + t]) : kk[(size_t)i * kc + t];
        cv[t] = emu ? bf16r(vv[(size_t)i * kc + t]) : vv[(size_t)i * kc + t];
      }
      if (emu)
        for (int t = 0; t < qc; ++t) q[(size_t)i * qc + t] = bf16r(q[(size_t)i * qc + t]);
    }
    if (last_q) return;
    // attention
    const float* Kl = cache.k + (size_t)l * cache.cap * kc;
    const float* Vl = cache.v + (size_t)l * cache.cap * kc;
#pragma omp parallel
    {
      std::vector<float> sc(cache.cap);
      std::vector<int> vis;
      vis.reserve(cache.cap);
#pragma omp for schedule(dynamic, 1)
      for (int i = 0; i < n; ++i) {
        vis.clear();
        for (int j = 0; j < cache.cap; ++j) {
          const bool ok = mask ? mask[(size_t)i * cache.cap + j] != 0
                               : (cache.pos[j] > 0 && cache.pos[j] <= positions[i]);
          if (ok) vis.push_back(j);
        }
        for (int hh = 0; hh < Hq; ++hh) {
          const float* qv = &q[(size_t)i * qc + hh * dh];
          const int hk = hh / G;
          float mx = -INFINITY;
          for (size_t t = 0; t < vis.size(); ++t) {
            const float* kr = Kl + (size_t)vis[t] * kc + hk * dh;
            float acc = 0.f;
#pragma omp simd reduction(+ : acc)
            for (int e = 0; e < dh; ++e) acc += qv[e] * kr[e];
            sc[t] = acc * scale;
            mx = std::max(mx, sc[t]);
          }
          double z = 0.0;
          for (size_t t = 0; t < vis.size(); ++t) {
            sc[t] = std::exp(sc[t] - mx);
            z += sc[t];
          }
          float* ov = &o[(size_t)i * qc + hh * dh];
          std::fill(ov, ov + dh, 0.f);
          const float inv = vis.empty() ? 0.f : (float)(1.0 / z);
          for (size_t t = 0; t < vis.size(); ++t) {
            const float* vr = Vl + (size_t)vis[t] * kc + hk * dh;
            const float w = sc[t] * inv;
#pragma omp simd
            for (int e = 0; e < dh; ++e) ov[e] += w * vr[e];
          }
          if (emu)
            for (int e = 0; e < dh; ++e) ov[e] = bf16r(ov[e]);
        }
      }
    }
    gemm_nt(o.data(), W.wo.data(), h.data(), n, d, qc, true);
    rmsnorm_rows(h.data(), W.ffn_norm.data(), x.data(), n, d, c.norm_eps, emu);
    gemm_nt(x.data(), W.wg.data(), gg.data(), n, F, d, false);
    gemm_nt(x.data(), W.wu.data(), uu.data(), n, F, d, false);
#pragma omp parallel for schedule(static)
    for (size_t t = 0; t < (size_t)n * F; ++t) {
      const float a = silu(gg[t]) * uu[t];
      gg[t] = emu ? bf16r(a) : a;
    }
    gemm_nt(gg.data(), W.wd.data(), h.data(), n, d, F, true);
  }
  if (logits && n_logit_rows > 0 && L == c.layers) {
    std::vector<float> hr((size_t)n_logit_rows * d), xr((size_t)n_logit_rows * d);
    for (int r = 0; r < n_logit_rows; ++r)
      std::memcpy(&hr[(size_t)r * d], &h[(size_t)logit_rows[r] * d], d * sizeof(float));
    rmsnorm_rows(hr.data(), m.final_norm.data(), xr.data(), n_logit_rows, d, c.norm_eps, emu);
    gemm_nt(xr.data(), m.lm_head.data(), logits, n_logit_rows, c.vocab, d, false);
  }
}

}  // namespace

// ============================================================================
extern "C" {

typedef struct orc_model orc_model;

// ---- Rng known-answer interface: kind 0 next_u64, 1 normal, 2 normal_f(0.02),
//      3 below(arg), 4 next_float, 5 next_double, 6 range(-arg, arg)
void orc_rng(uint64_t seed, int kind, int n, uint64_t arg, void* out) {
  Rng r(seed);
  for (int i = 0; i < n; ++i) {
    switch (kind) {
      case 0: static_cast<uint64_t*>(out)[i] = r.next_u64(); break;
      case 1: static_cast<double*>(out)[i] = r.normal(); break;
      case 2: static_cast<float*>(out)[i] = r.normal_f(0.02f); break;
      case 3: static_cast<uint64_t*>(out)[i] = r.below(arg); break;
      case 4: static_cast<float*>(out)[i] = r.next_float(); break;
      case 5: static_cast<double*>(out)[i] = r.next_double(); break;
      case 6: static_cast<int64_t*>(out)[i] = -(int64_t)arg + (int64_t)r.below(2 * arg + 1); break;
    }
  }
}

uint64_t orc_weight_seed(uint64_t seed, int tensor_id) {
  return mix64(seed + 0x9e3779b97f4a7c15ULL * (uint64_t)(tensor_id + 1));
}

// bf16(normal_f(sigma)) for every element of a [rows][cols] tensor drawn from
// Rng(stream_seed): sequential=1 runs the literal Rng (common.hpp:78-94);
// sequential=0 uses its counter form (pair j <- draws 2j, 2j+1), in parallel.
void orc_gen_normal(uint64_t stream_seed, size_t n, float sigma, int sequential, int round_bf16, float* out) {
  if (sequential) {
    Rng r(stream_seed);
    for (size_t i = 0; i < n; ++i) {
      const float v = r.normal_f(sigma);
      out[i] = round_bf16 ? bf16r(v) : v;
    }
    return;
  }
  const size_t pairs = (n + 1) / 2;
#pragma omp parallel for schedule(static)
  for (size_t j = 0; j < pairs; ++j) {
    const double u1 = (double)(splitmix_at(stream_seed, 2 * j) >> 11) * 0x1.0p-53;
    const double u2 = (double)(splitmix_at(stream_seed, 2 * j + 1) >> 11) * 0x1.0p-53;
    const double mag = std::sqrt(-2.0 * std::log(u1));
    const double e0 = mag * std::cos(6.283185307179586477 * u2);
    const double e1 = mag * std::sin(6.283185307179586477 * u2);
    const float f0 = (float)e0 * sigma, f1 = (float)e1 * sigma;
    out[2 * j] = round_bf16 ? bf16r(f0) : f0;
    if (2 * j + 1 < n) out[2 * j + 1] = round_bf16 ? bf16r(f1) : f1;
  }
}

void orc_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#endif
}
int orc_get_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

orc_model* orc_model_create(const orc_cfg* c) {
  auto* m = new Model();
  m->c = *c;
  const size_t d = c->d_model, V = c->vocab, F = c->ffn_dim, qc = (size_t)c->n_heads * c->head_dim,
               kc = (size_t)c->n_kv_heads * c->head_dim;
  m->emb.assign(V * d, 0.f);
  m->lm_head.assign(V * d, 0.f);
  m->final_norm.assign(d, 1.f);
  m->layers.resize(c->layers);
  for (auto& L : m->layers) {
    L.wq.assign(qc * d, 0.f);
    L.wk.assign(kc * d, 0.f);
    L.wv.assign(kc * d, 0.f);
    L.wo.assign(d * qc, 0.f);
    L.wg.assign(F * d, 0.f);
    L.wu.assign(F * d, 0.f);
    L.wd.assign(d * F, 0.f);
    L.attn_norm.assign(d, 1.f);
    L.ffn_norm.assign(d, 1.f);
  }
  m->theta.resize(c->head_dim / 2);
  for (int i = 0; i < c->head_dim / 2; ++i)
    m->theta[i] = std::pow(c->rope_base, -2.0 * (double)(i + 1) / (double)c->head_dim);
  return reinterpret_cast<orc_model*>(m);
}

void orc_model_free(orc_model* mm) { delete reinterpret_cast<Model*>(mm); }

// which: 0 emb 1 lm_head 2 wq 3 wk 4 wv 5 wo 6 w_gate 7 w_up 8 w_down 9 attn_norm 10 ffn_norm 11 final_norm
float* orc_model_tensor(orc_model* mm, int layer, int which, size_t* n_out) {
  Model* m = reinterpret_cast<Model*>(mm);
  std::vector<float>* t = nullptr;
  if (which == 0) t = &m->emb;
  else if (which == 1) t = &m->lm_head;
  else if (which == 11) t = &m->final_norm;
  else {
    if (layer < 0 || layer >= (int)m->layers.size()) return nullptr;
    Layer& L = m->layers[layer];
    std::vector<float>* tab[] = {nullptr, nullptr, &L.wq, &L.wk, &L.wv, &L.wo, &L.wg, &L.wu, &L.wd,
                                 &L.attn_norm, &L.ffn_norm};
    if (which < 2 || which > 10) return nullptr;
    t = tab[which];
  }
  if (n_out) *n_out = t->size();
  return t->data();
}

// init_model from the seed with the same tensor ids / streams as the GPU engine
// (paper_2601_12904_b200/csrc/engine.cpp): 0 emb, 1 lm_head, 16+8l+{0..6}.
void orc_model_init_seed(orc_model* mm, uint64_t seed) {
  Model* m = reinterpret_cast<Model*>(mm);
  const float sig = 0.02f;
  orc_gen_normal(orc_weight_seed(seed, 0), m->emb.size(), sig, 0, 1, m->emb.data());
  orc_gen_normal(orc_weight_seed(seed, 1), m->lm_head.size(), sig, 0, 1, m->lm_head.data());
  for (size_t l = 0; l < m->layers.size(); ++l) {
    Layer& L = m->layers[l];
    const int t0 = 16 + 8 * (int)l;
    std::vector<float>* ts[] = {&L.wq, &L.wk, &L.wv, &L.wo, &L.wg, &L.wu, &L.wd};
    for (int i = 0; i < 7; ++i) orc_gen_normal(orc_weight_seed(seed, t0 + i), ts[i]->size(), sig, 0, 1, ts[i]->data());
  }
}

// ---- rope
void orc_rope_apply(float* v, int dh, double pos, double base) {
  std::vector<double> th(dh / 2);
  for (int i = 0; i < dh / 2; ++i) th[i] = std::pow(base, -2.0 * (double)(i + 1) / (double)dh);
  rope_apply(v, dh, pos, th);
}
void orc_shift_rope(float* v, int dh, int old_pos, int new_pos, double base) {
  if (new_pos == old_pos) return;  // zero shift is the identity
  orc_rope_apply(v, dh, (double)new_pos - (double)old_pos, base);
}

// ---- forward (generic; see forward() above)
int orc_forward(const orc_model* mm, int n, const int32_t* tokens, const int32_t* positions, const int32_t* slots,
                float* cache_k, float* cache_v, int32_t* cache_pos, int cap, const uint8_t* mask, float* logits,
                int n_logit_rows, const int32_t* logit_rows, float* q_out, int stop_after_last_q, int emulate_bf16) {
  const Model* m = reinterpret_cast<const Model*>(mm);
  for (int i = 0; i < n; ++i) {
    if (tokens[i] < 0 || tokens[i] >= m->c.vocab) return 1;
    if (slots[i] < 0 || slots[i] >= cap) return 2;
    if (positions[i] < 1) return 3;
  }
  Cache c{cap, cache_k, cache_v, cache_pos};
  forward(*m, n, tokens, positions, slots, c, mask, logits, n_logit_rows, logit_rows, q_out, stop_after_last_q != 0,
          emulate_bf16 != 0);
  return 0;
}

// ---- stitch_full_reuse: fused = cat(KV_S, shifted chunks);
// chunk c lands at rows [dst_row_c, +n_c) with delta = target_start - native_start.
// Inputs/outputs [L][rows][Hkv][dh] fp32 (bf16-valued when round_bf16).
int orc_stitch(const orc_cfg* c, int n_chunks, const float* const* k_src, const float* const* v_src,
               const int32_t* n_tok, const int32_t* native_start, const int32_t* dst_row, float* k_out,
               float* v_out, int cap, int round_bf16) {
  const int kc = c->n_kv_heads * c->head_dim, dh = c->head_dim;
  std::vector<double> th(dh / 2);
  for (int i = 0; i < dh / 2; ++i) th[i] = std::pow(c->rope_base, -2.0 * (double)(i + 1) / (double)dh);
  for (int ch = 0; ch < n_chunks; ++ch) {
    const int delta = (dst_row[ch] + 1) - native_start[ch];
    std::vector<float> cs(dh);
    for (int i = 0; i < dh / 2; ++i) {
      const double a = (double)delta * th[i];
      cs[2 * i] = (float)std::cos(a);
      cs[2 * i + 1] = (float)std::sin(a);
    }
#pragma omp parallel for schedule(static)
    for (int l = 0; l < c->layers; ++l) {
      for (int t = 0; t < n_tok[ch]; ++t) {
        const float* ks = k_src[ch] + ((size_t)l * n_tok[ch] + t) * kc;
        const float* vs = v_src[ch] + ((size_t)l * n_tok[ch] + t) * kc;
        float* kd = k_out + ((size_t)l * cap + dst_row[ch] + t) * kc;
        float* vd = v_out + ((size_t)l * cap + dst_row[ch] + t) * kc;
        std::memcpy(vd, vs, kc * sizeof(float));
        if (delta == 0) {
          std::memcpy(kd, ks, kc * sizeof(float));
          continue;
        }
        for (int e = 0; e < kc; e += 2) {
          const int i = (e % dh) / 2;
          float o0, o1;
          rope_rotate_pair(ks[e], ks[e + 1], cs[2 * i], cs[2 * i + 1], o0, o1);
          kd[e] = round_bf16 ? bf16r(o0) : o0;
          kd[e + 1] = round_bf16 ? bf16r(o1) : o1;
        }
      }
    }
  }
  return 0;
}

// ---- select_query_guided scoring + argTopk.
// q [nq][Hq][dh] (final-layer, post-RoPE); keys [N][Hkv][dh] (final-layer stitched chunk keys).
// score[j] = sum_{t,h} softmax_j(q.k/sqrt(dh)) (joint over all N keys), or the raw-logit
// column sum when raw=1. sel: k indices (0-based into the N chunk keys),
// ascending; ties broken toward the lower index.
void orc_select(const float* q, const float* keys, int nq, int Hq, int Hkv, int dh, int N, int k, int raw,
                double* scores, int32_t* sel) {
  const int G = Hq / Hkv;
  const double scale = 1.0 / std::sqrt((double)dh);
  std::fill(scores, scores + N, 0.0);
  const int R = nq * Hq;
  std::vector<double> all((size_t)R * N);
#pragma omp parallel for schedule(static)
  for (int r = 0; r < R; ++r) {
    const int hh = r % Hq;
    const float* qv = q + (size_t)r * dh;
    double* row = &all[(size_t)r * N];
    double mx = -INFINITY;
    for (int j = 0; j < N; ++j) {
      const float* kv = keys + ((size_t)j * Hkv + hh / G) * dh;
      double acc = 0.0;
      for (int e = 0; e < dh; ++e) acc += (double)qv[e] * (double)kv[e];
      row[j] = acc * scale;
      mx = std::max(mx, row[j]);
    }
    if (!raw) {
      double z = 0.0;
      for (int j = 0; j < N; ++j) z += std::exp(row[j] - mx);
      for (int j = 0; j < N; ++j) row[j] = std::exp(row[j] - mx) / z;
    }
  }
#pragma omp parallel for schedule(static)
  for (int j = 0; j < N; ++j) {
    double s = 0.0;
    for (int r = 0; r < R; ++r) s += all[(size_t)r * N + j];
    scores[j] = s;
  }
  std::vector<int32_t> idx(N);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return scores[a] > scores[b]; });
  std::vector<int32_t> top(idx.begin(), idx.begin() + k);
  std::sort(top.begin(), top.end());
  std::copy(top.begin(), top.end(), sel);
}

// ---- q_sparse_attn, literal form of SPEC.md:153-161: shared cache is never
// written; fresh K/V of critical tokens live in exclusive pages (slot per
// critical token); query q_idx[i] attends every valid key at position <= its
// own, where stale positions read their exclusive-page entry instead.
// q [nq][H][dh]; shared K/V [T][H][dh] (single layer, MHA view); fresh [nq][H][dh]
// for all q indices (critical + new tokens); is_new[i] marks new-input tokens
// (appended logically after the shared region at their own positions).
int orc_q_sparse_attn(const float* q, const float* shared_k, const float* shared_v, int T, const float* fresh_k,
                      const float* fresh_v, const int32_t* q_idx, const uint8_t* is_new, int nq, int H, int dh,
                      float* out) {
  for (int i = 1; i < nq; ++i)
    if (q_idx[i] <= q_idx[i - 1]) return 1;  // plan invariant: strictly increasing
  const float scale = 1.0f / std::sqrt((float)dh);
  // exclusive page: slot of each critical (non-new) query index
  std::vector<int> page_of(T + 1, -1);
  for (int i = 0; i < nq; ++i)
    if (!is_new[i]) {
      if (q_idx[i] < 1 || q_idx[i] > T) return 2;  // plan references positions beyond shared_kv
      page_of[q_idx[i]] = i;
    }
#pragma omp parallel for schedule(dynamic, 1) collapse(2)
  for (int i = 0; i < nq; ++i) {
    for (int h = 0; h < H; ++h) {
      const int p = q_idx[i];
      std::vector<const float*> ks, vs;
      for (int pos = 1; pos <= std::min(p, T); ++pos) {
        const int pg = page_of[pos];
        if (pg >= 0) {  // stale original masked; fresh exclusive-page entry used
          ks.push_back(fresh_k + ((size_t)pg * H + h) * dh);
          vs.push_back(fresh_v + ((size_t)pg * H + h) * dh);
        } else {
          ks.push_back(shared_k + ((size_t)(pos - 1) * H + h) * dh);
          vs.push_back(shared_v + ((size_t)(pos - 1) * H + h) * dh);
        }
      }
      for (int j = 0; j < nq; ++j)  // new tokens at their own positions
        if (is_new[j] && q_idx[j] <= p) {
          ks.push_back(fresh_k + ((size_t)j * H + h) * dh);
          vs.push_back(fresh_v + ((size_t)j * H + h) * dh);
        }
      const float* qv = q + ((size_t)i * H + h) * dh;
      std::vector<double> s(ks.size());
      double mx = -INFINITY;
      for (size_t t = 0; t < ks.size(); ++t) {
        double a = 0.0;
        for (int e = 0; e < dh; ++e) a += (double)qv[e] * ks[t][e];
        s[t] = a * scale;
        mx = std::max(mx, s[t]);
      }
      double z = 0.0;
      for (auto& v : s) z += (v = std::exp(v - mx));
      float* o = out + ((size_t)i * H + h) * dh;
      for (int e = 0; e < dh; ++e) {
        double acc = 0.0;
        for (size_t t = 0; t < ks.size(); ++t) acc += s[t] * vs[t][e];
        o[e] = (float)(acc / z);
      }
    }
  }
  return 0;
}

// ---- build_equivalent_mask: dense [nq][T_total] visibility over the
// logical key list cat(shared[1..T], new tokens) with stale originals masked.
// key_pos[j]: position of logical key j; key_is_fresh[j]: 1 for fresh entries.
void orc_build_equivalent_mask(const int32_t* q_idx, const uint8_t* is_new, int nq, int T, uint8_t* mask) {
  // logical keys: shared positions 1..T (with critical ones replaced in place by their fresh entry)
  // followed by new-token entries; a query sees a key iff key position <= query position.
  const int n_new = (int)std::count(is_new, is_new + nq, 1);
  const int W = T + n_new;
  std::vector<int> kpos(W);
  for (int p = 1; p <= T; ++p) kpos[p - 1] = p;
  int w = T;
  for (int j = 0; j < nq; ++j)
    if (is_new[j]) kpos[w++] = q_idx[j];
  for (int i = 0; i < nq; ++i)
    for (int j = 0; j < W; ++j) mask[(size_t)i * W + j] = kpos[j] <= q_idx[i] ? 1 : 0;
}

// ---- kv_deviation (Eq. 7) over
// X = cat(S, chunks): Full Reuse = the stitched records (K1); Full Attention =
// KV_S (identical in both modes: prefix reuse, Eq. 4) followed by a prefill of
// every chunk token at its global position through the first n_layers layers.
// dev [N][n_layers][2] (fp64): sum over Hkv*dh of the squared K / V differences.
int orc_kv_deviation(const orc_model* mm, int S, const float* sys_k, const float* sys_v, int n_chunks,
                     const float* const* rec_k, const float* const* rec_v, const int32_t* const* rec_tok,
                     const int32_t* rec_n, const int32_t* rec_native, int n_layers, int emulate_bf16, double* dev) {
  const Model* m = reinterpret_cast<const Model*>(mm);
  const auto& c = m->c;
  if (n_layers < 1 || n_layers > c.layers) return 1;
  const int kc = c.n_kv_heads * c.head_dim;
  int N = 0;
  for (int i = 0; i < n_chunks; ++i) N += rec_n[i];
  const int cap = S + N;
  std::vector<float> fr_k((size_t)c.layers * cap * kc, 0.f), fr_v(fr_k.size(), 0.f);
  std::vector<const float*> ks, vs;
  std::vector<int32_t> ns, nat, dst;
  if (S > 0) {
    ks.push_back(sys_k), vs.push_back(sys_v), ns.push_back(S), nat.push_back(1), dst.push_back(0);
  }
  int row = S;
  for (int i = 0; i < n_chunks; ++i) {
    ks.push_back(rec_k[i]), vs.push_back(rec_v[i]), ns.push_back(rec_n[i]), nat.push_back(rec_native[i]);
    dst.push_back(row);
    row += rec_n[i];
  }
  orc_stitch(&c, (int)ks.size(), ks.data(), vs.data(), ns.data(), nat.data(), dst.data(), fr_k.data(), fr_v.data(),
             cap, emulate_bf16);
  // FA: system rows from KV_S, chunk rows prefilled at positions S+1..S+N
  std::vector<float> fa_k(fr_k.size(), 0.f), fa_v(fr_v.size(), 0.f);
  for (int l = 0; l < c.layers; ++l)
    for (int r = 0; r < S; ++r) {
      std::memcpy(&fa_k[((size_t)l * cap + r) * kc], &fr_k[((size_t)l * cap + r) * kc], kc * sizeof(float));
      std::memcpy(&fa_v[((size_t)l * cap + r) * kc], &fr_v[((size_t)l * cap + r) * kc], kc * sizeof(float));
    }
  std::vector<int32_t> pos(cap, 0), tok(N), p(N), sl(N);
  for (int r = 0; r < S; ++r) pos[r] = r + 1;
  {
    int off = 0;
    for (int i = 0; i < n_chunks; ++i) {
      std::memcpy(&tok[off], rec_tok[i], rec_n[i] * sizeof(int32_t));
      off += rec_n[i];
    }
  }
  for (int j = 0; j < N; ++j) p[j] = S + j + 1, sl[j] = S + j;
  Cache cc{cap, fa_k.data(), fa_v.data(), pos.data()};
  forward(*m, N, tok.data(), p.data(), sl.data(), cc, nullptr, nullptr, 0, nullptr, nullptr, true, emulate_bf16 != 0,
          n_layers);
#pragma omp parallel for schedule(static)
  for (int j = 0; j < N; ++j)
    for (int l = 0; l < n_layers; ++l) {
      const size_t o = ((size_t)l * cap + S + j) * kc;
      double dk = 0.0, dv = 0.0;
      for (int e = 0; e < kc; ++e) {
        const double a = (double)fa_k[o + e] - fr_k[o + e], b = (double)fa_v[o + e] - fr_v[o + e];
        dk += a * a;
        dv += b * b;
      }
      dev[((size_t)j * n_layers + l) * 2 + 0] = dk;
      dev[((size_t)j * n_layers + l) * 2 + 1] = dv;
    }
  return 0;
}

// ---- select_cacheblend (Eq. 8): argTopk of one deviation
// column (restricted to chunk tokens by construction), lower index on ties,
// returned ascending (0-based chunk-token indices).
void orc_select_cacheblend(const double* dev, int N, int n_layers, int layer, int comp, int k, int32_t* sel) {
  std::vector<double> v(N);
  for (int j = 0; j < N; ++j) {
    const double* d = dev + ((size_t)j * n_layers + (layer - 1)) * 2;
    v[j] = comp == 0 ? d[0] : (comp == 1 ? d[1] : d[0] + d[1]);
  }
  std::vector<int32_t> idx(N);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return v[a] > v[b]; });
  std::vector<int32_t> top(idx.begin(), idx.begin() + k);
  std::sort(top.begin(), top.end());
  std::copy(top.begin(), top.end(), sel);
}

// ---- full reprocess on one engine-shaped model.
// records: n_chunks chunk KV [L][n_c][Hkv][dh] fp32 at native_start_c; sys KV [L][S][Hkv][dh].
// Outputs: fused cache (cap >= T rows), logits of the last question row [V],
// crit positions (1-based, k of them), q_final [nq][Hq][dh], scores [N].
// inject: optional k critical positions (1-based) bypassing selection.
int orc_reprocess(const orc_model* mm, int S, const float* sys_k, const float* sys_v, const int32_t* sys_tok,
                  int n_chunks, const float* const* rec_k, const float* const* rec_v, const int32_t* const* rec_tok,
                  const int32_t* rec_n, const int32_t* rec_native, int nq, const int32_t* q_tok, float ratio,
                  int raw, const int32_t* inject, int n_inject, int emulate_bf16, float* k_cache, float* v_cache,
                  int cap, float* logits, int32_t* crit_out, int32_t* k_out, float* q_final, double* scores,
                  double* stage_seconds) {
  const Model* m = reinterpret_cast<const Model*>(mm);
  const auto& c = m->c;
  const int kc = c.n_kv_heads * c.head_dim;
  int N = 0;
  for (int i = 0; i < n_chunks; ++i) N += rec_n[i];
  const int T = S + N + nq;
  if (T > cap) return 1;
  auto now = []() {
#ifdef _OPENMP
    return omp_get_wtime();
#else
    return 0.0;
#endif
  };
  double t0 = now();
  std::vector<int32_t> pos(cap, 0);
  // 1. stitch (K1)
  {
    std::vector<const float*> ks, vs;
    std::vector<int32_t> ns, nat, dst;
    if (S > 0) {
      ks.push_back(sys_k);
      vs.push_back(sys_v);
      ns.push_back(S);
      nat.push_back(1);
      dst.push_back(0);
    }
    int row = S;
    for (int i = 0; i < n_chunks; ++i) {
      ks.push_back(rec_k[i]);
      vs.push_back(rec_v[i]);
      ns.push_back(rec_n[i]);
      nat.push_back(rec_native[i]);
      dst.push_back(row);
      row += rec_n[i];
    }
    orc_stitch(&c, (int)ks.size(), ks.data(), vs.data(), ns.data(), nat.data(), dst.data(), k_cache, v_cache, cap,
               emulate_bf16);
    for (int r = 0; r < S + N; ++r) pos[r] = r + 1;
  }
  double t1 = now();
  std::vector<int32_t> ctx_tok(N);
  {
    int off = 0;
    for (int i = 0; i < n_chunks; ++i) {
      std::memcpy(&ctx_tok[off], rec_tok[i], rec_n[i] * sizeof(int32_t));
      off += rec_n[i];
    }
  }
  // 2. question pass against the stitched cache, final-layer queries
  {
    std::vector<int32_t> qp(nq), qs(nq);
    for (int i = 0; i < nq; ++i) qs[i] = T - nq + i, qp[i] = T - nq + i + 1;
    Cache cc{cap, k_cache, v_cache, pos.data()};
    forward(*m, nq, q_tok, qp.data(), qs.data(), cc, nullptr, nullptr, 0, nullptr, q_final, true, emulate_bf16);
  }
  double t2 = now();
  // 3. selection
  int k = (int)std::floor((double)ratio * (double)N + 0.5);
  std::vector<int32_t> crit;
  if (inject) {
    k = n_inject;
    crit.assign(inject, inject + n_inject);
  } else {
    std::vector<float> keys((size_t)N * kc);
    for (int j = 0; j < N; ++j)
      std::memcpy(&keys[(size_t)j * kc], k_cache + ((size_t)(c.layers - 1) * cap + S + j) * kc, kc * sizeof(float));
    std::vector<int32_t> sel(std::max(k, 1));
    std::vector<double> sc(std::max(N, 1));
    if (N > 0) orc_select(q_final, keys.data(), nq, c.n_heads, c.n_kv_heads, c.head_dim, N, k, raw, sc.data(), sel.data());
    if (scores) std::copy(sc.begin(), sc.begin() + N, scores);
    for (int i = 0; i < k; ++i) crit.push_back(S + 1 + sel[i]);
  }
  double t3 = now();
  // 4. sparse prefill on QIndexPlan = crit U question, same index set every layer
  {
    const int M = k + nq;
    std::vector<int32_t> tok(M), p(M), sl(M);
    for (int i = 0; i < k; ++i) tok[i] = ctx_tok[crit[i] - S - 1], p[i] = crit[i], sl[i] = crit[i] - 1;
    for (int i = 0; i < nq; ++i) tok[k + i] = q_tok[i], p[k + i] = T - nq + i + 1, sl[k + i] = T - nq + i;
    int32_t last = M - 1;
    Cache cc{cap, k_cache, v_cache, pos.data()};
    forward(*m, M, tok.data(), p.data(), sl.data(), cc, nullptr, logits, 1, &last, nullptr, false, emulate_bf16);
  }
  double t4 = now();
  if (crit_out) std::copy(crit.begin(), crit.end(), crit_out);
  if (k_out) *k_out = k;
  if (stage_seconds) {
    stage_seconds[0] = t1 - t0;
    stage_seconds[1] = t2 - t1;
    stage_seconds[2] = t3 - t2;
    stage_seconds[3] = t4 - t3;
  }
  (void)sys_tok;
  return 0;
}

}  // extern "C"
