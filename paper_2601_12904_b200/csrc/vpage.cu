// Shared V pages (§4.3):
// a request's V rows stay in the store's records, only the rows it computes
// (critical, question, decoded) live in its exclusive region. This file holds
// the per-request patch plan the attention kernels follow (vpatch_plan) and
// the read-back that materialises the fused V view (vpage_gather).
//
// Plan, per sequence, over 128-row key tiles of its cache rows: the primary
// segment of tile j holds row 128j (its TMA box supplies every row of that
// record in the tile, zeros elsewhere); the entries list, in row order, each
// row the box gets wrong -- a row of another segment (chunk boundary, KV_S) or
// a fresh critical row (exclusive slot = crit_slot0 + its rank among the
// critical rows = its GEMM row). Rows >= tail_row0 (question / decoded rows)
// are fresh by rule and never listed.
#include "kernels.h"
#include "ptx.cuh"

namespace fragk {

namespace {

constexpr int VP_THREADS = 1024;

// exclusive block-wide prefix sum of one value per thread; returns the total
__device__ int block_exclusive_scan(int v, int* red, int& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) red[w] = x;
  __syncthreads();
  if (w == 0) {
    int s = lane < (int)(blockDim.x >> 5) ? red[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    red[lane] = s;  // inclusive warp totals
  }
  __syncthreads();
  const int before = (w > 0 ? red[w - 1] : 0) + x - v;
  total = red[(blockDim.x >> 5) - 1];
  __syncthreads();
  return before;
}

// last segment with row0 <= row, -1 if row is in no segment
__device__ __forceinline__ int seg_of(const int* s_row0, const int* s_n, int n_seg, int row) {
  int lo = 0, hi = n_seg - 1, f = -1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    if (s_row0[mid] <= row) {
      f = mid;
      lo = mid + 1;
    } else {
      hi = mid - 1;
    }
  }
  return (f >= 0 && row < s_row0[f] + s_n[f]) ? f : -1;
}

__global__ void __launch_bounds__(VP_THREADS) vpatch_plan_kernel(const VPlanArgs* __restrict__ seqs) {
  const VPlanArgs A = seqs[blockIdx.x];
  extern __shared__ int sm[];
  __shared__ int red[32];
  const int W = (A.n_rows + 31) >> 5;
  const int tiles = (A.n_rows + 127) >> 7;
  uint32_t* bits = reinterpret_cast<uint32_t*>(sm);  // [W] fresh critical rows
  int* wpre = sm + W;                                  // [W] exclusive popcount prefix
  int* tcnt = wpre + W;                                // [tiles]
  int* s_row0 = tcnt + tiles;                          // [n_seg]
  int* s_n = s_row0 + A.n_seg;                         // [n_seg]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < A.n_seg; i += VP_THREADS) {
    s_row0[i] = A.segs[i].row0;
    s_n[i] = A.segs[i].n;
  }
  for (int w = tid; w < W; w += VP_THREADS) bits[w] = 0u;
  pdl_wait();  // the critical rows come from the preceding top-k
  pdl_launch_dependents();
  __syncthreads();
  for (int i = tid; i < A.n_crit; i += VP_THREADS) {
    const int row = A.crit[i] - A.row_base;
    if (row >= 0 && row < A.n_rows && row < A.tail_row0) atomicOr(&bits[row >> 5], 1u << (row & 31));
  }
  __syncthreads();
  {  // exclusive popcount prefix over the bitmap words (contiguous word range per thread)
    const int per = (W + VP_THREADS - 1) / VP_THREADS;
    const int lo = min(W, tid * per), hi = min(W, lo + per);
    int c = 0;
    for (int w = lo; w < hi; ++w) c += __popc(bits[w]);
    int total;
    int run = block_exclusive_scan(c, red, total);
    for (int w = lo; w < hi; ++w) {
      wpre[w] = run;
      run += __popc(bits[w]);
    }
  }
  __syncthreads();
  // row decision: 0 = the box has it (or nobody needs it), else the entry
  auto entry = [&](int row, int key0, int prim) -> unsigned long long {
    if (row >= A.n_rows || row >= A.tail_row0) return 0ull;
    const uint32_t wbits = bits[row >> 5];
    const uint32_t b = 1u << (row & 31);
    const unsigned long long rin = (unsigned long long)(row - key0);
    if (wbits & b) {
      const int slot = A.crit_slot0 + wpre[row >> 5] + __popc(wbits & (b - 1u));
      return rin | ((unsigned long long)(uint32_t)slot << 32) | (1ull << 7);  // bit 7: non-empty marker
    }
    const int s = seg_of(s_row0, s_n, A.n_seg, row);
    if (s < 0 || s == prim) return 0ull;
    return rin | ((unsigned long long)(s + 1) << 8) | ((unsigned long long)(uint32_t)(row - s_row0[s]) << 32) |
           (1ull << 7);
  };
  // pass 1: entries per tile (one warp per tile, 4 rows per lane)
  for (int t = warp; t < tiles; t += VP_THREADS / 32) {
    const int key0 = t << 7;
    const int prim = seg_of(s_row0, s_n, A.n_seg, key0);
    int c = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) c += __popc(__ballot_sync(0xffffffffu, entry(key0 + q * 32 + lane, key0, prim) != 0ull));
    if (lane == 0) tcnt[t] = c;
  }
  __syncthreads();
  {  // tile starts
    const int per = (tiles + VP_THREADS - 1) / VP_THREADS;
    const int lo = min(tiles, tid * per), hi = min(tiles, lo + per);
    int c = 0;
    for (int t = lo; t < hi; ++t) c += tcnt[t];
    int total;
    int run = block_exclusive_scan(c, red, total);
    for (int t = lo; t < hi; ++t) {
      A.vtile[t] = run;
      const int n = tcnt[t];
      tcnt[t] = run;
      run += n;
    }
    if (tid == 0) A.vtile[tiles] = total;
  }
  __syncthreads();
  // pass 2: entries in row order + the tile's TMA source
  for (int t = warp; t < tiles; t += VP_THREADS / 32) {
    const int key0 = t << 7;
    const int prim = seg_of(s_row0, s_n, A.n_seg, key0);
    int off = tcnt[t];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const unsigned long long e = entry(key0 + q * 32 + lane, key0, prim);
      const uint32_t ball = __ballot_sync(0xffffffffu, e != 0ull);
      if (e) A.vent[off + __popc(ball & ((1u << lane) - 1u))] = e & ~(1ull << 7);
      off += __popc(ball);
    }
    // no primary: segment 0 at a row past its end (all-zero box)
    if (lane == 0) A.vprim[t] = prim >= 0 ? make_int2(prim, key0 - s_row0[prim]) : make_int2(0, s_n[0]);
  }
}

// Read-back: fused V rows [0, n_rows) of every layer (grid: tiles x layers).
__global__ void __launch_bounds__(256) vpage_gather_kernel(const VSeg* __restrict__ segs, const int* __restrict__ vtile,
                                                           const int2* __restrict__ vprim,
                                                           const unsigned long long* __restrict__ vent,
                                                           const bf16* __restrict__ vx, size_t vx_ls, int tail_row0,
                                                           int tail_slot0, int n_rows, int kvc, bf16* __restrict__ dst,
                                                           size_t dst_ls) {
  __shared__ const bf16* src[128];
  const int tile = blockIdx.x, l = blockIdx.y, key0 = tile * 128;
  const int2 pr = vprim[tile];
  if (threadIdx.x < 128) {
    const int row = key0 + threadIdx.x;
    const bf16* p = nullptr;
    if (row < n_rows) {
      if (row >= tail_row0) {
        p = vx + l * vx_ls + (size_t)(tail_slot0 + row - tail_row0) * kvc;
      } else {
        const VSeg& s = segs[pr.x];
        const int y = pr.y + (int)threadIdx.x;
        if (y < s.n) p = s.v + ((size_t)l * s.n + y) * kvc;
      }
    }
    src[threadIdx.x] = p;
  }
  __syncthreads();
  for (int e = vtile[tile] + (int)threadIdx.x; e < vtile[tile + 1]; e += blockDim.x) {
    const unsigned long long ent = vent[e];
    const int r = (int)(ent & 127);
    const int sg = (int)((ent >> 8) & 0xffffff);
    const size_t srow = (size_t)(ent >> 32);
    src[r] = sg == 0 ? vx + l * vx_ls + srow * kvc : segs[sg - 1].v + ((size_t)l * segs[sg - 1].n + srow) * kvc;
  }
  __syncthreads();
  const int nv = kvc / 8;  // 16-byte vectors per row
  for (int i = threadIdx.x; i < 128 * nv; i += blockDim.x) {
    const int r = i / nv, c = i - r * nv;
    if (key0 + r >= n_rows) continue;
    const uint4 v = src[r] ? reinterpret_cast<const uint4*>(src[r])[c] : make_uint4(0u, 0u, 0u, 0u);
    reinterpret_cast<uint4*>(dst + l * dst_ls + (size_t)(key0 + r) * kvc)[c] = v;
  }
}

// one CTA row-slice per (segment, row block): 16-byte streaming copy
__global__ void __launch_bounds__(256) vwindow_fill_kernel(const VSeg* __restrict__ segs, int layer, int kvc,
                                                           bf16* __restrict__ dst) {
  const VSeg& g = segs[blockIdx.y];
  const int nv = kvc / 8;
  const long total = (long)g.n * nv;
  const uint4* src = reinterpret_cast<const uint4*>(g.v + (size_t)layer * g.n * kvc);
  uint4* out = reinterpret_cast<uint4*>(dst + (size_t)(g.base + g.row0) * kvc);
  pdl_launch_dependents();
  const long stride = (long)gridDim.x * blockDim.x;
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < total; i += 4 * stride) {  // the window is read by the attention after the next GEMM
    const uint4 a0 = ld_stream(src + i), a1 = ld_stream(src + i + stride);
    const uint4 a2 = ld_stream(src + i + 2 * stride), a3 = ld_stream(src + i + 3 * stride);
    out[i] = a0;
    out[i + stride] = a1;
    out[i + 2 * stride] = a2;
    out[i + 3 * stride] = a3;
  }
  for (; i < total; i += stride) out[i] = ld_stream(src + i);
}

}  // namespace

int vwindow_fill(const VSeg* segs, int n_seg, int max_rows, int layer, int kvc, bf16* dst, cudaStream_t stream) {
  if (n_seg <= 0 || max_rows <= 0) return 0;
  if (kvc % 8) return -1;
  const long vecs = (long)max_rows * (kvc / 8);
  long bx = (vecs + 4 * 256 - 1) / (4 * 256);
  const long cap = (long)num_sms() * 8 / (n_seg < 8 ? n_seg : 8) + 1;
  if (bx > cap) bx = cap;
  if (bx < 1) bx = 1;
  vwindow_fill_kernel<<<dim3((unsigned)bx, (unsigned)n_seg), 256, 0, stream>>>(segs, layer, kvc, dst);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

static size_t vpatch_plan_smem(int max_rows, int max_segs) {
  const size_t W = ((size_t)max_rows + 31) / 32, tiles = ((size_t)max_rows + 127) / 128;
  return (2 * W + tiles + 2 * (size_t)max_segs) * sizeof(int);
}

bool vpatch_plan_fits(int max_rows, int max_segs) { return vpatch_plan_smem(max_rows, max_segs) <= 227 * 1024 - 256; }

int vpatch_plan(const VPlanArgs* seqs_dev, int n_seq, int max_rows, int max_segs, cudaStream_t stream) {
  if (n_seq <= 0) return 0;
  const size_t smem = vpatch_plan_smem(max_rows, max_segs);
  if (!vpatch_plan_fits(max_rows, max_segs)) return -1;
  if (smem > 48 * 1024) smem_attr_once(vpatch_plan_kernel, (int)(227 * 1024));
  launch_pdl(vpatch_plan_kernel, dim3(n_seq), dim3(VP_THREADS), smem, stream, seqs_dev);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int vpage_gather(const VSeg* segs, const int* vtile, const int2* vprim, const unsigned long long* vent,
                 const bf16* vx, size_t vx_layer_stride, int tail_row0, int tail_slot0, int n_rows, int L, int kvc,
                 bf16* dst, size_t dst_layer_stride, cudaStream_t stream) {
  if (n_rows <= 0 || L <= 0) return 0;
  if (kvc % 8) return -1;
  dim3 grid((unsigned)((n_rows + 127) / 128), (unsigned)L);
  vpage_gather_kernel<<<grid, 256, 0, stream>>>(segs, vtile, vprim, vent, vx, vx_layer_stride, tail_row0, tail_slot0,
                                                n_rows, kvc, dst, dst_layer_stride);
  return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace fragk
