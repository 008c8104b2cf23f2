// K6: sparse-Q causal attention over the fused KV cache (SPEC.md:153-161,
// SPEC.md:177-178; PAPER.md:691-704 Q-index sparse attention).
//
// Only the selected query rows (critical tokens + question, ascending fused
// rows p_i) are computed. Row i attends to fused rows [0, p_i]: the per-request
// fused cache already holds this layer's fresh K/V at every selected row
// (scattered by the QKV epilogue), so stale entries are replaced and earlier
// critical tokens' fresh K/V are visible within the same pass,
// while the store's records are never touched.
//
// v1 kernel: FlashAttention-2 style with mma.sync m16n8k16 (bf16 in, fp32
// accumulate), online softmax in registers, cp.async double-buffered K/V tiles
// of 64 keys shared by all query heads of one GQA group (64 query rows per CTA =
// 64/G tokens x G heads), and optional split-KV with an LSE combine pass.
#include <cfloat>

#include "kernels.h"
#include "ptx.cuh"

namespace fragk {

namespace {

constexpr int ATT_ROWS = 64;   // query rows per CTA (4 warps x 16)
constexpr int ATT_KEYS = 64;   // keys per tile
constexpr int ATT_THREADS = 128;

__device__ __forceinline__ void cp_async16(uint32_t smem, const void* gmem, bool valid) {
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Swizzled byte offset of 16-byte chunk c of key row r in a [64][DH] bf16 tile.
template <int DH>
__device__ __forceinline__ uint32_t tile_off(int r, int c) {
  return (uint32_t)(r * DH * 2 + ((c ^ (r & 7)) << 4));
}

template <int DH>
__global__ void __launch_bounds__(ATT_THREADS) attn_kernel(const AttnArgs a, int G, int n_qblocks) {
  constexpr int CH = DH / 8;  // 16-byte chunks per key row
  constexpr int TILE_BYTES = ATT_KEYS * DH * 2;
  extern __shared__ __align__(128) uint8_t sm[];
  uint8_t* sK = sm;                    // [2][64][DH]
  uint8_t* sV = sm + 2 * TILE_BYTES;   // [2][64][DH]

  const int qb = n_qblocks - 1 - (int)blockIdx.x;  // heaviest (latest rows) first
  const int hk = blockIdx.y;
  const int split = blockIdx.z;
  const int tok_per_cta = ATT_ROWS / G;
  const int t0 = qb * tok_per_cta;
  const int t_end = min(t0 + tok_per_cta, a.M);
  const int warp = warp_id(), lane = lane_id();
  const int g = lane >> 2, tq = lane & 3;

  const int p_max = a.rows[t_end - 1];
  const int p_min = a.rows[t0];
  const int k_lo = a.n_splits > 1 ? split * a.split_keys : 0;
  int k_hi = p_max + 1;
  if (a.n_splits > 1) k_hi = min(k_hi, (split + 1) * a.split_keys);

  // rows of this thread: r0 = 16*warp + g, r1 = r0 + 8
  int tok[2], head[2], prow[2];
  bool live[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int r = 16 * warp + g + 8 * i;
    tok[i] = t0 + r / G;
    head[i] = hk * G + r % G;
    live[i] = tok[i] < a.M;
    prow[i] = live[i] ? a.rows[tok[i]] : -1;
  }

  const size_t kv_row_stride = (size_t)a.Hkv * DH;
  auto out_write = [&](float (&o)[DH / 8][4], float (&m)[2], float (&l)[2]) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      if (!live[i]) continue;
      const size_t qi = (size_t)tok[i] * a.Hq + head[i];
      if (a.n_splits > 1) {
        float* po = a.part_o + ((size_t)split * a.M * a.Hq + qi) * DH;
        const float inv = l[i] > 0.f ? 1.f / l[i] : 0.f;
#pragma unroll
        for (int nt = 0; nt < DH / 8; ++nt)
          *reinterpret_cast<float2*>(po + nt * 8 + 2 * tq) = make_float2(o[nt][2 * i] * inv, o[nt][2 * i + 1] * inv);
        if (tq == 0)
          a.part_lse[(size_t)split * a.M * a.Hq + qi] = l[i] > 0.f ? m[i] + __logf(l[i]) : -INFINITY;
      } else {
        bf16* po = a.out + qi * DH;
        const float inv = l[i] > 0.f ? 1.f / l[i] : 0.f;
#pragma unroll
        for (int nt = 0; nt < DH / 8; ++nt)
          *reinterpret_cast<uint32_t*>(po + nt * 8 + 2 * tq) = pack_bf16(o[nt][2 * i] * inv, o[nt][2 * i + 1] * inv);
      }
    }
  };

  float o[DH / 8][4];
#pragma unroll
  for (int nt = 0; nt < DH / 8; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};

  if (k_lo >= k_hi) {  // this split lies beyond every row of the block
    out_write(o, m, l);
    return;
  }

  // Q fragments (A operand, 16 rows x DH) straight from global.
  uint32_t qf[DH / 16][4];
  {
    const bf16* q0 = a.q + ((size_t)tok[0] * a.Hq + head[0]) * DH;
    const bf16* q1 = a.q + ((size_t)tok[1] * a.Hq + head[1]) * DH;
#pragma unroll
    for (int kk = 0; kk < DH / 16; ++kk) {
      const int c = kk * 16 + 2 * tq;
      qf[kk][0] = live[0] ? *reinterpret_cast<const uint32_t*>(q0 + c) : 0u;
      qf[kk][1] = live[1] ? *reinterpret_cast<const uint32_t*>(q1 + c) : 0u;
      qf[kk][2] = live[0] ? *reinterpret_cast<const uint32_t*>(q0 + c + 8) : 0u;
      qf[kk][3] = live[1] ? *reinterpret_cast<const uint32_t*>(q1 + c + 8) : 0u;
    }
  }

  const bf16* kbase = a.k + (size_t)hk * DH;
  const bf16* vbase = a.v + (size_t)hk * DH;
  auto load_tile = [&](int buf, int key0) {
    const uint32_t kdst = smem_u32(sK + buf * TILE_BYTES);
    const uint32_t vdst = smem_u32(sV + buf * TILE_BYTES);
#pragma unroll
    for (int it = 0; it < (ATT_KEYS * CH) / ATT_THREADS; ++it) {
      const int idx = it * ATT_THREADS + threadIdx.x;
      const int r = idx / CH, c = idx % CH;
      const int key = key0 + r;
      const bool ok = key < a.T;
      const size_t off = (size_t)(ok ? key : 0) * kv_row_stride + c * 8;
      cp_async16(kdst + tile_off<DH>(r, c), kbase + off, ok);
      cp_async16(vdst + tile_off<DH>(r, c), vbase + off, ok);
    }
    cp_async_commit();
  };

  const float sl2 = a.scale * 1.4426950408889634f;
  const int n_tiles = (k_hi - k_lo + ATT_KEYS - 1) / ATT_KEYS;
  load_tile(0, k_lo);
  for (int it = 0; it < n_tiles; ++it) {
    const int key0 = k_lo + it * ATT_KEYS;
    if (it + 1 < n_tiles) {
      load_tile((it + 1) & 1, key0 + ATT_KEYS);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const uint32_t kt = smem_u32(sK + (it & 1) * TILE_BYTES);
    const uint32_t vt = smem_u32(sV + (it & 1) * TILE_BYTES);

    // S = Q K^T : 16 rows x 64 keys per warp.
    float s[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int k2 = 0; k2 < DH / 32; ++k2) {
        // matrices: dims [32k2 + 8j, +8) for j = lane/8, keys 8nt + lane%8
        const int r = nt * 8 + (lane & 7);
        const int c = k2 * 4 + (lane >> 3);
        uint32_t b0, b1, b2, b3;
        ldsm_x4(kt + tile_off<DH>(r, c), b0, b1, b2, b3);
        mma16816(s[nt], qf[2 * k2], b0, b1);
        mma16816(s[nt], qf[2 * k2 + 1], b2, b3);
      }
    }
    // causal mask by position + split bound
    const bool need_mask = (key0 + ATT_KEYS - 1 > p_min) || (key0 + ATT_KEYS > k_hi);
    if (need_mask) {
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int key = key0 + nt * 8 + 2 * tq + (e & 1);
          const int i = e >> 1;
          if (key > prow[i] || key >= k_hi) s[nt][e] = -INFINITY;
        }
      }
    }
    // online softmax (rows g and g+8; a row is spread over the 4 threads of a quad)
    float mnew[2], corr[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      float mx = m[i];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) mx = fmaxf(mx, fmaxf(s[nt][2 * i], s[nt][2 * i + 1]));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      mnew[i] = mx;
      corr[i] = (m[i] == -INFINITY) ? 0.f : exp2f((m[i] - mx) * sl2);
      m[i] = mx;
    }
    float rs[2] = {0.f, 0.f};
    uint32_t pf[4][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      float p[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = e >> 1;
        p[e] = (mnew[i] == -INFINITY) ? 0.f : exp2f((s[nt][e] - mnew[i]) * sl2);
      }
      rs[0] += p[0] + p[1];
      rs[1] += p[2] + p[3];
      const int kk = nt >> 1, hi = nt & 1;
      pf[kk][2 * hi + 0] = pack_bf16(p[0], p[1]);
      pf[kk][2 * hi + 1] = pack_bf16(p[2], p[3]);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      rs[i] += __shfl_xor_sync(0xffffffffu, rs[i], 1);
      rs[i] += __shfl_xor_sync(0xffffffffu, rs[i], 2);
      l[i] = l[i] * corr[i] + rs[i];
    }
#pragma unroll
    for (int nt = 0; nt < DH / 8; ++nt) {
      o[nt][0] *= corr[0];
      o[nt][1] *= corr[0];
      o[nt][2] *= corr[1];
      o[nt][3] *= corr[1];
    }
    // O += P V : A = P (16 x 64 keys), B = V (64 keys x DH)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t af[4] = {pf[kk][0], pf[kk][1], pf[kk][2], pf[kk][3]};
#pragma unroll
      for (int n2 = 0; n2 < DH / 16; ++n2) {
        // matrices: (keys 16kk + 8*(j&1), dims 16n2 + 8*(j>>1)), j = lane/8
        const int j = lane >> 3;
        const int r = kk * 16 + (j & 1) * 8 + (lane & 7);
        const int c = n2 * 2 + (j >> 1);
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(vt + tile_off<DH>(r, c), b0, b1, b2, b3);
        mma16816(o[2 * n2], af, b0, b1);
        mma16816(o[2 * n2 + 1], af, b2, b3);
      }
    }
    __syncthreads();
  }
  // l holds the quad-reduced row sum; m the running max (in raw-score units).
  float mm[2] = {m[0] * sl2 / 1.4426950408889634f, m[1] * sl2 / 1.4426950408889634f};
  out_write(o, mm, l);
}

// Merge split partials: out = sum_s w_s O_s / sum_s w_s, w_s = exp(lse_s - max).
template <int DH>
__global__ void attn_combine_kernel(const AttnArgs a) {
  const size_t qi = blockIdx.x;  // (token, head)
  const size_t MH = (size_t)a.M * a.Hq;
  float mx = -INFINITY;
  for (int s = 0; s < a.n_splits; ++s) mx = fmaxf(mx, a.part_lse[s * MH + qi]);
  const int d = threadIdx.x;  // DH threads
  float acc = 0.f, wsum = 0.f;
  for (int s = 0; s < a.n_splits; ++s) {
    const float lse = a.part_lse[s * MH + qi];
    if (lse == -INFINITY) continue;
    const float w = __expf(lse - mx);
    wsum += w;
    acc += w * a.part_o[(s * MH + qi) * DH + d];
  }
  a.out[qi * DH + d] = __float2bfloat16_rn(wsum > 0.f ? acc / wsum : 0.f);
}

}  // namespace

int sparse_q_attention(const AttnArgs& a0, cudaStream_t stream) {
  AttnArgs a = a0;
  if (a.M <= 0) return 0;
  const int G = a.Hq / a.Hkv;
  if (G <= 0 || ATT_ROWS % G != 0 || a.Hq % a.Hkv != 0) return -1;
  const int tok_per_cta = ATT_ROWS / G;
  const int n_qblocks = (a.M + tok_per_cta - 1) / tok_per_cta;
  if (a.split_keys <= 0 || a.n_splits <= 1) {
    a.n_splits = 1;
  }
  dim3 grid(n_qblocks, a.Hkv, a.n_splits);
  int launches = 0;
  if (a.dh == 128) {
    const int smem = 4 * ATT_KEYS * 128 * 2;
    cudaFuncSetAttribute(attn_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attn_kernel<128><<<grid, ATT_THREADS, smem, stream>>>(a, G, n_qblocks);
    ++launches;
    if (a.n_splits > 1) {
      attn_combine_kernel<128><<<(unsigned)((size_t)a.M * a.Hq), 128, 0, stream>>>(a);
      ++launches;
    }
  } else if (a.dh == 64) {
    const int smem = 4 * ATT_KEYS * 64 * 2;
    attn_kernel<64><<<grid, ATT_THREADS, smem, stream>>>(a, G, n_qblocks);
    ++launches;
    if (a.n_splits > 1) {
      attn_combine_kernel<64><<<(unsigned)((size_t)a.M * a.Hq), 64, 0, stream>>>(a);
      ++launches;
    }
  } else {
    return -1;
  }
  return launches;
}

}  // namespace fragk
