// K2 — SAGE mean aggregation (forward) and its transpose (backward), the
// readout backward, K4 pooling, and deterministic column reductions.
//
//   forward   m[v]  = (1/deg v) * sum_{u->v} h[u]            gnn.py:157-158, 206
//   backward  dh[u] = dA_self[u] + sum_{u->v} dA_neigh[v]/deg v  gnn.py:161-162, 232
//   readout   dh3[v] = dr[g(v)] / N_g                          gnn.py:224
//   pool      u[g]  = [mean_{v in g} h3[v], (fs-mu)/sigma]     gnn.py:214-215, 96-97
//
// Layout: node rows are contiguous per graph (graph_ptr), activation rows are
// 16-byte aligned and processed 8 columns per lane with 128-bit loads.  All
// reductions run in a fixed order (no float atomics): results are
// bit-reproducible run to run.
#include <algorithm>

#include "common.cuh"

namespace dippm {

constexpr int kAggThreads = 256;
constexpr int kAggColCap = 2048;   // neighbour ids staged in shared memory per block
constexpr int kColsumRows = 64;    // rows per block for column partial sums
constexpr int kColsumGroup = 64;   // block partials folded per level-2 partial (fused bias-gradient reduce)

__host__ __device__ inline int colsum_groups(int nblk) { return (nblk + kColsumGroup - 1) / kColsumGroup; }

// Both aggregation kernels stage the block's slice of the CSR (row pointers,
// neighbour ids, 1/deg weights) in shared memory first, so the per-row work is
// only independent 128-bit feature-row loads (no dependent index loads on the
// critical path), and each lane keeps CPL 8-column chunks x 2 neighbours in
// flight.  A warp covers one row when width/8 >= 32 (hidden 512: 2 chunks per
// lane), or 32/L rows for narrow layers (layer 1, width 32).
constexpr int kRowsPerBlock = 64;
// agg^T / readout kernels with the fused bias reduction: up to this many rows per block, so
// the grid is one wave of resident blocks (their per-block barrier / fold tail is amortised
// over more rows per warp)
constexpr int kRowsPerBlockT = 256;

template <int DT, int CPL>
__device__ __forceinline__ void load_chunks(const ActView& a, int64_t r, int c0, int stride, float (&x)[CPL][8]) {
#pragma unroll
  for (int q = 0; q < CPL; ++q) act_load8_t<DT>(a, r, c0 + q * stride, x[q]);
}

// Forward: m[v] = (1/deg v) * sum_{u->v} h[u]; optionally self_out[v] = h[v].
// DTI: dtype of h (fp32 X for layer 1, the compute dtype after), DTO: of m.
template <int DTI, int DTO, int CPL>
__global__ void __launch_bounds__(kAggThreads, 4) k_aggregate(ActView h, ActView m, ActView self_out, int64_t N,
                                                              int rpb, int width, const int* __restrict__ rowptr,
                                                              const int* __restrict__ col,
                                                              const float* __restrict__ inv_deg) {
  __shared__ int s_ptr[kRowsPerBlockT + 1];
  __shared__ float s_w[kRowsPerBlockT];
  __shared__ int s_col[kAggColCap];
  pdl_begin();
  const int L = (width >> 3) / CPL;  // lanes per row
  const int gpw = 32 / L;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / L, sub = lane % L;
  const int64_t r0 = (int64_t)blockIdx.x * rpb;
  const int nrows = (int)((N - r0 < rpb) ? N - r0 : rpb);
  const int cbeg = rowptr[r0];
  for (int i = threadIdx.x; i <= nrows; i += blockDim.x) s_ptr[i] = rowptr[r0 + i] - cbeg;
  for (int i = threadIdx.x; i < nrows; i += blockDim.x) s_w[i] = inv_deg[r0 + i];
  const int ncol = rowptr[r0 + nrows] - cbeg;
  const bool staged = ncol <= kAggColCap;
  if (staged)
    for (int i = threadIdx.x; i < ncol; i += blockDim.x) s_col[i] = col[cbeg + i];
  __syncthreads();
  if (grp >= gpw) return;
  const int c0 = sub * 8, stride = L * 8;
  const int rstep = (kAggThreads / 32) * gpw;
  // bf16 rows: the next row's first neighbour is fetched (raw) while this row is summed, so
  // each warp keeps two rows' loads in flight
  uint4 nxt[CPL];
  auto fetch_first = [&](int lr2) {
    if constexpr (DTI == DIPPM_DT_BF16) {
      if (lr2 < nrows && s_ptr[lr2] < s_ptr[lr2 + 1]) {
        const int v = staged ? s_col[s_ptr[lr2]] : col[cbeg + s_ptr[lr2]];
        const __nv_bfloat16* src = reinterpret_cast<const __nv_bfloat16*>(h.base) + (int64_t)v * h.ld + c0;
#pragma unroll
        for (int q = 0; q < CPL; ++q) nxt[q] = __ldg(reinterpret_cast<const uint4*>(src + q * stride));
      }
    }
  };
  fetch_first(warp * gpw + grp);
  for (int lr = warp * gpw + grp; lr < nrows; lr += rstep) {
    const int64_t row = r0 + lr;
    const int b = s_ptr[lr], e = s_ptr[lr + 1];
    float acc[CPL][8] = {};
    float xs[CPL][8];
    if constexpr (DTI == DIPPM_DT_F32) {
      // layer 1: the row's own features (copied next to the mean) and its first two neighbours
      // are loaded before any of them is used, one memory latency per row for the common
      // in-degrees; pairs are summed in CSR order
      if (self_out.base) load_chunks<DTI, CPL>(h, row, c0, stride, xs);
      int j = b;
      for (; j + 1 < e; j += 2) {
        float x0[CPL][8], x1[CPL][8];
        load_chunks<DTI, CPL>(h, staged ? s_col[j] : col[cbeg + j], c0, stride, x0);
        load_chunks<DTI, CPL>(h, staged ? s_col[j + 1] : col[cbeg + j + 1], c0, stride, x1);
#pragma unroll
        for (int q = 0; q < CPL; ++q)
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            acc[q][k] += x0[q][k];
            acc[q][k] += x1[q][k];
          }
      }
      if (j < e) {
        float x[CPL][8];
        load_chunks<DTI, CPL>(h, staged ? s_col[j] : col[cbeg + j], c0, stride, x);
#pragma unroll
        for (int q = 0; q < CPL; ++q)
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[q][k] += x[q][k];
      }
    } else if constexpr (DTI == DIPPM_DT_BF16) {
      uint4 cur[CPL];
#pragma unroll
      for (int q = 0; q < CPL; ++q) cur[q] = nxt[q];
      fetch_first(lr + rstep);
      if (b < e) {  // first neighbour (prefetched), then the rest in CSR order
#pragma unroll
        for (int q = 0; q < CPL; ++q) {
          const __nv_bfloat162* hh = reinterpret_cast<const __nv_bfloat162*>(&cur[q]);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 f = __bfloat1622float2(hh[i]);
            acc[q][2 * i] += f.x;
            acc[q][2 * i + 1] += f.y;
          }
        }
      }
      for (int j = b + 1; j < e; ++j) {
        float x[CPL][8];
        load_chunks<DTI, CPL>(h, staged ? s_col[j] : col[cbeg + j], c0, stride, x);
#pragma unroll
        for (int q = 0; q < CPL; ++q)
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[q][k] += x[q][k];
      }
    } else {
      for (int j = b; j < e; ++j) {
        float x[CPL][8];
        load_chunks<DTI, CPL>(h, staged ? s_col[j] : col[cbeg + j], c0, stride, x);
#pragma unroll
        for (int q = 0; q < CPL; ++q)
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[q][k] += x[q][k];
      }
    }
    const float w = s_w[lr];
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[q][k] *= w;
      act_store8_t<DTO>(m, row, c0 + q * stride, acc[q]);
    }
    if (self_out.base) {
      if constexpr (DTI != DIPPM_DT_F32) load_chunks<DTI, CPL>(h, row, c0, stride, xs);
#pragma unroll
      for (int q = 0; q < CPL; ++q) act_store8_t<DTO>(self_out, row, c0 + q * stride, xs[q]);
    }
  }
}

// Transposed aggregation for the backward pass (gnn.py:161-162, 232): with
// B = [dz | g] ([N, 2*width], dz already in the left half),
//   g[u] = sum_{u->v} dz[v] / deg(v)          (agg^T dz, via the transposed CSR)
// so that dh_prev = [dz | g] @ [W_self | W_neigh]^T is ONE GEMM (dgrad with the
// ReLU gate fused in its epilogue).  Also emits per-block column partial sums
// of dz (bias gradient, gnn.py:230), reduced over the block's row slots in a
// fixed order.  write_agg = 0: partial sums only.
// kReadout: layer 3 — dz3 is not materialised yet; it is formed on the fly from
// the readout gradient (gnn.py:224, 227): dz3[v] = du[g(v)] / N_g * (h3[v] > 0),
// written into B's left half while g = agg^T dz3 goes to the right half.  All
// neighbours of v lie in v's graph, so one graph id per row suffices.
// out[c] = sum_{r0 <= r < r1} x[r*width + c] for all c < width, by one block:
// thread t owns 4 columns (float4) of one of `halves` row ranges, 8 L2 loads in
// flight; the range sums are combined in range order through shared memory.
// Fixed order throughout (fp64), so the result is deterministic.
__device__ __forceinline__ void fold_rows_block(const float* x, int r0, int r1, int width, float* out,
                                                double* s_fold /* [kAggThreads * 4] */) {
  const int c4n = width >> 2;
  const int halves = (int)blockDim.x / c4n;  // width 512: 2 row ranges of 128 column groups
  const int t = threadIdx.x, h = t / c4n, c = (t % c4n) * 4;
  double a[4] = {0.0, 0.0, 0.0, 0.0};
  if (h < halves) {
    const int n = r1 - r0;
    const int lo = r0 + h * n / halves, hi = r0 + (h + 1) * n / halves;
    int r = lo;
    for (; r + 8 <= hi; r += 8) {
      float4 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = __ldcg(reinterpret_cast<const float4*>(x + (int64_t)(r + k) * width + c));
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        a[0] += v[k].x; a[1] += v[k].y; a[2] += v[k].z; a[3] += v[k].w;
      }
    }
    for (; r < hi; ++r) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(x + (int64_t)r * width + c));
      a[0] += v.x; a[1] += v.y; a[2] += v.z; a[3] += v.w;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) s_fold[h * width + c + k] = a[k];
  }
  __syncthreads();
  for (int cc = threadIdx.x; cc < width; cc += blockDim.x) {
    double tot = 0.0;
    for (int q = 0; q < halves; ++q) tot += s_fold[q * width + cc];
    out[cc] = (float)tot;
  }
}

struct ReadoutArgs {
  const float* du;          // [G, ld_du] fp32 (dr = du[:, :width])
  int64_t ld_du;
  const int* graph_ptr;     // [G+1]
  const int* node_graph;    // [N]
  ActView h3;               // ReLU gate (values), used when h3_bits is NULL
  const uint32_t* h3_bits;  // 1-bit (h3 > 0) masks from the layer-3 forward epilogue, word [(c/32)*bits_ld + r]
                            // (bits_ld 0: row-major, word [r*(width/32) + c/32])
  int64_t bits_ld;
  int64_t width_words;      // width / 32 (row-major bit masks)
};

// ReLU'(z3) for 8 consecutive columns per chunk: from the forward's bit mask (4 bytes per 32
// columns) when present, else by reading h3 (z > 0 <=> h > 0).
template <int DT, int CPL>
__device__ __forceinline__ void relu_gate(const ReadoutArgs& ro, int64_t r, int c0, int stride, bool (&gt)[CPL][8]) {
  if (ro.h3_bits) {
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      const int c = c0 + q * stride;
      const uint32_t w = __ldg(ro.bits_ld ? ro.h3_bits + (int64_t)(c >> 5) * ro.bits_ld + r
                                          : ro.h3_bits + r * (int64_t)(ro.width_words) + (c >> 5)) >> (c & 31);
#pragma unroll
      for (int k = 0; k < 8; ++k) gt[q][k] = (w >> k) & 1u;
    }
  } else {
    float hg[CPL][8];
    load_chunks<DT, CPL>(ro.h3, r, c0, stride, hg);
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
      for (int k = 0; k < 8; ++k) gt[q][k] = hg[q][k] > 0.f;
  }
}

// Fused bias-gradient reduction (gnn.py:230) after a block has written its column partial:
// two fixed-order levels — the last block of each group of kColsumGroup blocks folds the
// group's partials (block order) into a level-2 row, the last group folds those (group
// order) into bias_out.  Counters return to zero.  s_scratch: >= 8 KB of shared memory.
__device__ __forceinline__ void finish_bias(float* colsum_partial, int width, float* bias_out, int* sync,
                                            float* s_scratch) {
    // Fused bias-gradient reduction (gnn.py:230), two fixed-order levels: the last
    // block of each group of kColsumGroup blocks folds the group's partials (in
    // block order) into a level-2 row; the last group to finish folds those (in
    // group order) into bias_out.  Counters return to zero for the next launch.
    __shared__ int s_last;
    const int nblk = (int)gridDim.x, ngroups = colsum_groups(nblk);
    const int grp = blockIdx.x / kColsumGroup;
    float* l2 = colsum_partial + (int64_t)nblk * width;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const int gsize = min(kColsumGroup, nblk - grp * kColsumGroup);
      s_last = atomicAdd(&sync[grp], 1) == gsize - 1;
    }
    __syncthreads();
    if (!s_last) return;
    const int b0 = grp * kColsumGroup, b1 = min(nblk, b0 + kColsumGroup);
    double* s_fold = reinterpret_cast<double*>(s_scratch);  // the warp partials are no longer needed
    fold_rows_block(colsum_partial, b0, b1, width, l2 + (int64_t)grp * width, s_fold);
    __syncthreads();
    if (threadIdx.x == 0) {
      sync[grp] = 0;
      __threadfence();
      s_last = atomicAdd(&sync[ngroups], 1) == ngroups - 1;
    }
    __syncthreads();
    if (!s_last) return;
    fold_rows_block(l2, 0, ngroups, width, bias_out, s_fold);
    if (threadIdx.x == 0) sync[ngroups] = 0;
}

template <int DT, int CPL, bool kReadout>
__global__ void __launch_bounds__(kAggThreads, kReadout ? 2 : 3) k_aggregate_t(ActView B, int width, int64_t N,
                                                                               int rpb, int write_agg,
                                                                const int* __restrict__ t_rowptr,
                                                                const int* __restrict__ t_col,
                                                                const float* __restrict__ inv_deg,
                                                                float* __restrict__ colsum_partial, ReadoutArgs ro,
                                                                float* __restrict__ bias_out, int* __restrict__ sync) {
  extern __shared__ float s_part[];  // [8 warps * gpw][width]
  __shared__ int s_ptr[kRowsPerBlockT + 1];
  __shared__ int s_col[kAggColCap];
  __shared__ float s_cw[kAggColCap];
  pdl_begin();
  const int L = (width >> 3) / CPL;
  const int gpw = 32 / L;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / L, sub = lane % L;
  const int64_t r0 = (int64_t)blockIdx.x * rpb;
  const int nrows = (int)((N - r0 < rpb) ? N - r0 : rpb);
  const int cbeg = t_rowptr[r0];
  const int ncol = t_rowptr[r0 + nrows] - cbeg;
  const bool staged = ncol <= kAggColCap;
  __shared__ int s_g[kRowsPerBlockT];  // readout: graph of each row of the block
  if (write_agg) {
    for (int i = threadIdx.x; i <= nrows; i += blockDim.x) s_ptr[i] = t_rowptr[r0 + i] - cbeg;
    if (staged)
      for (int i = threadIdx.x; i < ncol; i += blockDim.x) {
        const int v = t_col[cbeg + i];
        s_col[i] = v;
        s_cw[i] = inv_deg[v];
      }
    if constexpr (kReadout)
      for (int i = threadIdx.x; i < nrows; i += blockDim.x) s_g[i] = ro.node_graph[r0 + i];
    __syncthreads();
  }
  const int c0 = sub * 8, stride = L * 8;
  float part[CPL][8] = {};
  float dr[CPL][8];  // readout: du[g(row)] / N_g (shared by the row and its neighbours), kept while g repeats
  int g_cur = -1;
  if (grp < gpw) {
    for (int lr = warp * gpw + grp; lr < nrows; lr += (kAggThreads / 32) * gpw) {
      const int64_t row = r0 + lr;
      float own[CPL][8];
      if constexpr (kReadout) {
        const int g = s_g[lr];
        if (g != g_cur) {  // rows of a graph are contiguous: reload only at graph changes
          g_cur = g;
          const float inv_n = 1.0f / (float)(ro.graph_ptr[g + 1] - ro.graph_ptr[g]);
          const float* dp = ro.du + (int64_t)g * ro.ld_du;
#pragma unroll
          for (int q = 0; q < CPL; ++q) {
            const float4 a = __ldg(reinterpret_cast<const float4*>(dp + c0 + q * stride));
            const float4 b2 = __ldg(reinterpret_cast<const float4*>(dp + c0 + q * stride + 4));
            dr[q][0] = a.x * inv_n; dr[q][1] = a.y * inv_n; dr[q][2] = a.z * inv_n; dr[q][3] = a.w * inv_n;
            dr[q][4] = b2.x * inv_n; dr[q][5] = b2.y * inv_n; dr[q][6] = b2.z * inv_n; dr[q][7] = b2.w * inv_n;
          }
        }
        bool gt[CPL][8];
        relu_gate<DT, CPL>(ro, row, c0, stride, gt);
#pragma unroll
        for (int q = 0; q < CPL; ++q) {
#pragma unroll
          for (int k = 0; k < 8; ++k) own[q][k] = gt[q][k] ? dr[q][k] : 0.f;
          act_store8_t<DT>(B, row, c0 + q * stride, own[q]);
        }
      } else {
        load_chunks<DT, CPL>(B, row, c0, stride, own);
      }
      if (write_agg) {
        const int b = s_ptr[lr], e = s_ptr[lr + 1];
        float acc[CPL][8] = {};
        for (int j = b; j < e; ++j) {
          const int v0 = staged ? s_col[j] : t_col[cbeg + j];
          const float w0 = staged ? s_cw[j] : inv_deg[v0];
          float x[CPL][8];
          if constexpr (kReadout) {
            bool gt[CPL][8];
            relu_gate<DT, CPL>(ro, v0, c0, stride, gt);
#pragma unroll
            for (int q = 0; q < CPL; ++q)
#pragma unroll
              for (int k = 0; k < 8; ++k) x[q][k] = gt[q][k] ? dr[q][k] : 0.f;
          } else {
            load_chunks<DT, CPL>(B, v0, c0, stride, x);
          }
#pragma unroll
          for (int q = 0; q < CPL; ++q)
#pragma unroll
            for (int k = 0; k < 8; ++k) acc[q][k] = fmaf(w0, x[q][k], acc[q][k]);
        }
#pragma unroll
        for (int q = 0; q < CPL; ++q) act_store8_t<DT>(B, row, width + c0 + q * stride, acc[q]);
      }
#pragma unroll
      for (int q = 0; q < CPL; ++q)
#pragma unroll
        for (int k = 0; k < 8; ++k) part[q][k] += own[q][k];
    }
    const int slot = warp * gpw + grp;
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
      for (int k = 0; k < 8; ++k) s_part[slot * width + c0 + q * stride + k] = part[q][k];
  }
  __syncthreads();
  const int slots = (kAggThreads / 32) * gpw;
  for (int c = threadIdx.x; c < width; c += blockDim.x) {
    float t = 0.f;
    for (int q = 0; q < slots; ++q) t += s_part[q * width + c];
    colsum_partial[(int64_t)blockIdx.x * width + c] = t;
  }
  if (bias_out) finish_bias(colsum_partial, width, bias_out, sync, s_part);
  else if (sync && blockIdx.x == 0 && threadIdx.x == 0) *sync = (int)gridDim.x;  // deferred fold: the row count
}

// Layer-3 readout backward gated by the forward's bit masks (the fast path of
// dippm_readout_aggregate_t):  dz3[v, c] = dr[g, c] * bit(v, c) with dr = du[g] / N_g, and
// since every neighbour of u lies in u's graph,
//   (agg^T dz3)[u, c] = dr[g, c] * sum_{u->v} bit(v, c) / deg(v).
// The block first stages the bit words of its own rows plus a halo of kBitsHalo rows past
// them (operator graphs are topologically ordered, so out-neighbours are mostly a few rows
// ahead) in shared memory with one burst of coalesced loads; the per-row work is then
// shared-memory reads and 128-bit stores, with a global load only for a neighbour outside
// the staged window.  One warp per row, CPL chunks of 8 columns per lane.
constexpr int kBitsHalo = 64;
template <int DT, int CPL>
__global__ void __launch_bounds__(kAggThreads, CPL >= 3 ? 2 : 3) k_readout_agg_bits(ActView B, int width, int64_t N, int rpb,
                                                                     const int* __restrict__ t_rowptr,
                                                                     const int* __restrict__ t_col,
                                                                     const float* __restrict__ inv_deg,
                                                                     float* __restrict__ colsum_partial, ReadoutArgs ro,
                                                                     float* __restrict__ bias_out,
                                                                     int* __restrict__ sync) {
  extern __shared__ float s_part[];  // [8 warps][width] floats, then the staged bit words
  __shared__ int s_ptr[kRowsPerBlockT + 1];
  __shared__ int s_col[kAggColCap];
  __shared__ float s_cw[kAggColCap];
  __shared__ int s_g[kRowsPerBlockT];
  pdl_begin();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * rpb;
  const int nrows = (int)((N - r0 < rpb) ? N - r0 : rpb);
  const int cbeg = t_rowptr[r0];
  const int ncol = t_rowptr[r0 + nrows] - cbeg;
  const bool staged = ncol <= kAggColCap;
  // word of (row, chunk): chunk-major (stride bits_ld per chunk) or row-major (stride 1)
  const int64_t cstride = ro.bits_ld ? ro.bits_ld : 1, rstride = ro.bits_ld ? 1 : width >> 5;
  const int W = width >> 5;
  const int R = (int)((N - r0 < rpb + kBitsHalo) ? N - r0 : rpb + kBitsHalo);  // staged rows [r0, r0 + R)
  uint32_t* s_bits = reinterpret_cast<uint32_t*>(s_part + (kAggThreads / 32) * width);  // [W][R]
  for (int i = threadIdx.x; i < W * R; i += blockDim.x) {
    const int w = i / R, r = i - w * R;
    s_bits[i] = __ldg(ro.h3_bits + w * cstride + (r0 + r) * rstride);
  }
  for (int i = threadIdx.x; i <= nrows; i += blockDim.x) s_ptr[i] = t_rowptr[r0 + i] - cbeg;
  for (int i = threadIdx.x; i < nrows; i += blockDim.x) s_g[i] = ro.node_graph[r0 + i];
  if (staged)
    for (int i = threadIdx.x; i < ncol; i += blockDim.x) {
      const int v = t_col[cbeg + i];
      s_col[i] = v;
      s_cw[i] = inv_deg[v];
    }
  __syncthreads();
  const int stride = 32 * 8;  // a warp covers one row: lane chunks c0 = 8*lane + q*256
  const int c0 = lane * 8;
  int wofs[CPL], wsh[CPL];  // word index (column chunk) and bit offset of each of the lane's chunks
#pragma unroll
  for (int q = 0; q < CPL; ++q) {
    wofs[q] = (c0 + q * stride) >> 5;
    wsh[q] = (c0 + q * stride) & 31;
  }
  float part[CPL][8] = {};
  float dr[CPL][8];
  int g_cur = -1;
  for (int lr = warp; lr < nrows; lr += kAggThreads / 32) {
    const int64_t row = r0 + lr;
    const int b = s_ptr[lr], e = s_ptr[lr + 1];
    const int g = s_g[lr];
    if (g != g_cur) {  // rows of a graph are contiguous: reload dr only at graph changes
      g_cur = g;
      const float inv_n = 1.0f / (float)(ro.graph_ptr[g + 1] - ro.graph_ptr[g]);
      const float* dp = ro.du + (int64_t)g * ro.ld_du;
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(dp + c0 + q * stride));
        const float4 a2 = __ldg(reinterpret_cast<const float4*>(dp + c0 + q * stride + 4));
        dr[q][0] = a.x * inv_n; dr[q][1] = a.y * inv_n; dr[q][2] = a.z * inv_n; dr[q][3] = a.w * inv_n;
        dr[q][4] = a2.x * inv_n; dr[q][5] = a2.y * inv_n; dr[q][6] = a2.z * inv_n; dr[q][7] = a2.w * inv_n;
      }
    }
    float acc[CPL][8] = {};
    for (int j = b; j < e; ++j) {  // out-edges in CSR order
      const int v0 = staged ? s_col[j] : t_col[cbeg + j];
      const float w0 = staged ? s_cw[j] : inv_deg[v0];
      const unsigned rel = (unsigned)(v0 - r0);
      uint32_t wv[CPL];
#pragma unroll
      for (int q = 0; q < CPL; ++q)
        wv[q] = (rel < (unsigned)R ? s_bits[wofs[q] * R + rel] : __ldg(ro.h3_bits + wofs[q] * cstride + (int64_t)v0 * rstride)) >> wsh[q];
#pragma unroll
      for (int q = 0; q < CPL; ++q)
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[q][k] += (wv[q] >> k) & 1u ? w0 : 0.f;
    }
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      float own[8];
      const uint32_t wo = s_bits[wofs[q] * R + lr] >> wsh[q];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        own[k] = (wo >> k) & 1u ? dr[q][k] : 0.f;
        part[q][k] += own[k];
        acc[q][k] *= dr[q][k];
      }
      act_store8_t<DT>(B, row, c0 + q * stride, own);
      act_store8_t<DT>(B, row, width + c0 + q * stride, acc[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < CPL; ++q)
#pragma unroll
    for (int k = 0; k < 8; ++k) s_part[warp * width + c0 + q * stride + k] = part[q][k];
  __syncthreads();
  for (int c = threadIdx.x; c < width; c += blockDim.x) {
    float t = 0.f;
    for (int q = 0; q < kAggThreads / 32; ++q) t += s_part[q * width + c];
    colsum_partial[(int64_t)blockIdx.x * width + c] = t;
  }
  if (bias_out) finish_bias(colsum_partial, width, bias_out, sync, s_part);
  else if (sync && blockIdx.x == 0 && threadIdx.x == 0) *sync = (int)gridDim.x;  // deferred fold: the row count
}

// The training step's layout of the same computation (bf16 B, row-major bit masks,
// width = 256 * CPL): one row's CPL*8 bit words are contiguous, so the block's rows plus the
// halo are staged with 16-byte copies in the row-major order the warps read them (a lane's
// words for its chunks are a broadcast LDS each); the neighbour loop has no layout or
// dtype generality, the first neighbour initialises the accumulator, and the rare
// neighbour outside the staged window / block with more than kAggColCap out-edges takes a
// separate uniform branch; a row with one out-edge (the common case) forms dr * w0 * bit
// directly.  At configs[1] the row loop runs at the write bandwidth (29 us for 157 MB against
// 27 us for a bare store loop of the same pattern); the rest of the launch is the staging
// prologue and the bias fold.
template <int CPL>
__global__ void __launch_bounds__(kAggThreads, CPL >= 3 ? 2 : 4) k_readout_bits_rm(__nv_bfloat16* __restrict__ Bp, int64_t ldb,
                                                                    int64_t N, int rpb,
                                                                    const int* __restrict__ t_rowptr,
                                                                    const int* __restrict__ t_col,
                                                                    const float* __restrict__ inv_deg,
                                                                    float* __restrict__ colsum_partial,
                                                                    ReadoutArgs ro, float* __restrict__ bias_out,
                                                                    int* __restrict__ sync) {
  constexpr int W = CPL * 8;  // bit words per row
  constexpr int width = CPL * 256;
  extern __shared__ __align__(16) float s_part[];  // [8 warps][width], then the staged bit words [R][W]
  __shared__ int s_ptr[kRowsPerBlockT + 1];
  __shared__ int s_col[kAggColCap];
  __shared__ float s_cw[kAggColCap];
  __shared__ int s_g[kRowsPerBlockT];
  pdl_begin();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * rpb;
  const int nrows = (int)((N - r0 < rpb) ? N - r0 : rpb);
  const int R = (int)((N - r0 < rpb + kBitsHalo) ? N - r0 : rpb + kBitsHalo);
  const int cbeg = t_rowptr[r0];
  const int ncol = t_rowptr[r0 + nrows] - cbeg;
  const bool staged = ncol <= kAggColCap;
  uint32_t* s_bits = reinterpret_cast<uint32_t*>(s_part + (kAggThreads / 32) * width);
  {
    const uint4* src = reinterpret_cast<const uint4*>(ro.h3_bits + r0 * W);
    uint4* dst = reinterpret_cast<uint4*>(s_bits);
    for (int i = threadIdx.x; i < R * (W / 4); i += blockDim.x) dst[i] = __ldg(src + i);
  }
  for (int i = threadIdx.x; i <= nrows; i += blockDim.x) s_ptr[i] = t_rowptr[r0 + i] - cbeg;
  for (int i = threadIdx.x; i < nrows; i += blockDim.x) s_g[i] = ro.node_graph[r0 + i];
  if (staged)
    for (int i = threadIdx.x; i < ncol; i += blockDim.x) {
      const int v = t_col[cbeg + i];
      s_col[i] = v;
      s_cw[i] = inv_deg[v];
    }
  __syncthreads();
  const int c0 = lane * 8;            // lane chunks: columns c0 + q * 256 .. + 8
  const int wl = lane >> 2, sh = (lane & 3) * 8;  // word (of each 256-column group) and bit offset
  float part[CPL][8] = {};
  float dr[CPL][8];
  int g_cur = -1;
  // bit words of neighbour v (staged window, else global)
  auto nbits = [&](int v, uint32_t (&wv)[CPL]) {
    const unsigned rel = (unsigned)((int64_t)v - r0);
    if (rel < (unsigned)R) {
#pragma unroll
      for (int q = 0; q < CPL; ++q) wv[q] = s_bits[rel * W + q * 8 + wl] >> sh;
    } else {
#pragma unroll
      for (int q = 0; q < CPL; ++q) wv[q] = __ldg(ro.h3_bits + (int64_t)v * W + q * 8 + wl) >> sh;
    }
  };
  auto rows = [&](auto staged_tag) {
    constexpr bool kStaged = decltype(staged_tag)::value;
    for (int lr = warp; lr < nrows; lr += kAggThreads / 32) {
      const int b = s_ptr[lr], e = s_ptr[lr + 1];
      const int g = s_g[lr];
      if (g != g_cur) {  // rows of a graph are contiguous: reload dr only at graph changes
        g_cur = g;
        const float inv_n = 1.0f / (float)(ro.graph_ptr[g + 1] - ro.graph_ptr[g]);
        const float* dp = ro.du + (int64_t)g * ro.ld_du;
#pragma unroll
        for (int q = 0; q < CPL; ++q) {
          const float4 a = __ldg(reinterpret_cast<const float4*>(dp + c0 + q * 256));
          const float4 a2 = __ldg(reinterpret_cast<const float4*>(dp + c0 + q * 256 + 4));
          dr[q][0] = a.x * inv_n; dr[q][1] = a.y * inv_n; dr[q][2] = a.z * inv_n; dr[q][3] = a.w * inv_n;
          dr[q][4] = a2.x * inv_n; dr[q][5] = a2.y * inv_n; dr[q][6] = a2.z * inv_n; dr[q][7] = a2.w * inv_n;
        }
      }
      __nv_bfloat16* brow = Bp + (r0 + lr) * ldb + c0;
      // own rows: dz3 = dr * bit (and the bias partial)
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const uint32_t x = s_bits[lr * W + q * 8 + wl] >> sh;
        uint4 o;
        uint32_t* op = &o.x;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float o0 = (x >> (2 * i)) & 1u ? dr[q][2 * i] : 0.f;
          const float o1 = (x >> (2 * i + 1)) & 1u ? dr[q][2 * i + 1] : 0.f;
          part[q][2 * i] += o0;
          part[q][2 * i + 1] += o1;
          __nv_bfloat162 ho = __floats2bfloat162_rn(o0, o1);
          op[i] = *reinterpret_cast<uint32_t*>(&ho);
        }
        *reinterpret_cast<uint4*>(brow + q * 256) = o;
      }
      // agg^T dz3 = dr * sum_{u->v} bit(v) / deg(v); one out-edge (the common case): dr * w0 * bit
      uint4 ag[CPL];
      if (e - b == 1) {
        const int v = kStaged ? s_col[b] : t_col[cbeg + b];
        const float w0 = kStaged ? s_cw[b] : inv_deg[v];
        uint32_t wv[CPL];
        nbits(v, wv);
#pragma unroll
        for (int q = 0; q < CPL; ++q) {
          uint32_t* ap = &ag[q].x;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float a0 = (wv[q] >> (2 * i)) & 1u ? w0 * dr[q][2 * i] : 0.f;
            const float a1 = (wv[q] >> (2 * i + 1)) & 1u ? w0 * dr[q][2 * i + 1] : 0.f;
            __nv_bfloat162 ha = __floats2bfloat162_rn(a0, a1);
            ap[i] = *reinterpret_cast<uint32_t*>(&ha);
          }
        }
      } else {
        float acc[CPL][8];
#pragma unroll
        for (int q = 0; q < CPL; ++q)
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[q][k] = 0.f;
        for (int j = b; j < e; ++j) {  // out-edges in CSR order
          const int v = kStaged ? s_col[j] : t_col[cbeg + j];
          const float w0 = kStaged ? s_cw[j] : inv_deg[v];
          uint32_t wv[CPL];
          nbits(v, wv);
#pragma unroll
          for (int q = 0; q < CPL; ++q)
#pragma unroll
            for (int k = 0; k < 8; ++k) acc[q][k] += (wv[q] >> k) & 1u ? w0 : 0.f;
        }
#pragma unroll
        for (int q = 0; q < CPL; ++q) {
          uint32_t* ap = &ag[q].x;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            __nv_bfloat162 ha = __floats2bfloat162_rn(acc[q][2 * i] * dr[q][2 * i], acc[q][2 * i + 1] * dr[q][2 * i + 1]);
            ap[i] = *reinterpret_cast<uint32_t*>(&ha);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < CPL; ++q) *reinterpret_cast<uint4*>(brow + width + q * 256) = ag[q];
    }
  };
  if (staged) rows(std::true_type{});
  else rows(std::false_type{});
#pragma unroll
  for (int q = 0; q < CPL; ++q)
#pragma unroll
    for (int k = 0; k < 8; ++k) s_part[warp * width + c0 + q * 256 + k] = part[q][k];
  __syncthreads();
  for (int c = threadIdx.x; c < width; c += blockDim.x) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < kAggThreads / 32; ++w) t += s_part[w * width + c];
    colsum_partial[(int64_t)blockIdx.x * width + c] = t;
  }
  if (bias_out) finish_bias(colsum_partial, width, bias_out, sync, s_part);
  else if (sync && blockIdx.x == 0 && threadIdx.x == 0) *sync = (int)gridDim.x;  // deferred fold: the row count
}

// Readout backward (gnn.py:224, 227): dz3[v] = du[g(v), :width] / N_g * (h3[v] > 0).
__global__ void __launch_bounds__(kAggThreads) k_readout_backward(const float* __restrict__ du, int64_t ld_du,
                                                                  int width, ActView gate, ActView dz, int64_t N,
                                                                  const int* __restrict__ graph_ptr, int64_t G) {
  const int chunks = width >> 3;
  const int groups = kAggThreads / chunks;
  const int grp = threadIdx.x / chunks, ch = threadIdx.x % chunks;
  const int64_t r0 = (int64_t)blockIdx.x * kColsumRows;
  const int64_t r1 = (N < r0 + kColsumRows) ? N : r0 + kColsumRows;
  if (grp >= groups || r0 + grp >= r1) return;
  const int c = ch * 8;
  int lo = 0, hi = (int)G;  // graph of the first row handled by this thread
  const int64_t rr = r0 + grp;
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (graph_ptr[mid] <= rr) lo = mid; else hi = mid;
  }
  int g = lo;
  for (int64_t row = rr; row < r1; row += groups) {
    while (graph_ptr[g + 1] <= row) ++g;
    const float inv_n = 1.0f / (float)(graph_ptr[g + 1] - graph_ptr[g]);
    const float* p = du + (int64_t)g * ld_du + c;
    float v[8], hg[8];
    act_load8(gate, row, c, hg);
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = hg[k] > 0.f ? __ldg(p + k) * inv_n : 0.f;  // relu'(z): z>0 <=> h>0
    act_store8(dz, row, c, v);
  }
}

// Deterministic column reduction: out[c] = scale * sum_r in[r*ld + c].
// 32 columns x 32 row-lanes per block, fixed-order fp64 accumulation.
__global__ void __launch_bounds__(1024) k_reduce_rows(const float* __restrict__ in, int64_t rows, int64_t ld,
                                                      int cols, double scale, float* __restrict__ out) {
  __shared__ double s[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + tx;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;  // independent chains: 4 loads in flight
  if (c < cols) {
    int64_t r = ty;
    for (; r + 96 < rows; r += 128) {
      a0 += (double)in[r * ld + c];
      a1 += (double)in[(r + 32) * ld + c];
      a2 += (double)in[(r + 64) * ld + c];
      a3 += (double)in[(r + 96) * ld + c];
    }
    for (; r < rows; r += 32) a0 += (double)in[r * ld + c];
  }
  s[ty][tx] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  if (ty == 0 && c < cols) {
    double t = 0.0;
    for (int q = 0; q < 32; ++q) t += s[q][tx];
    out[c] = (float)(t * scale);
  }
}

// K4: one block per graph (16 warps); a warp reads a whole h3 row with
// 128-bit loads (CPL chunks of 8 columns per lane), rows strided over the warps,
// then a fixed-order smem reduction over warps.  u = [mean_g h3 | (fs-mu)/sigma | 0]
// in the head's operand dtype, row stride u.ld (>= width + 5, zero padded).
constexpr int kPoolThreads = 512;
template <int DT, int CPL>
__global__ void __launch_bounds__(kPoolThreads) k_pool_concat(ActView h, const int* __restrict__ graph_ptr,
                                                              int width, const double* __restrict__ fs_raw,
                                                              const double* __restrict__ norm, ActView u) {
  extern __shared__ float s_part[];  // [slots][width]
  const int g = blockIdx.x;
  const int L = (width >> 3) / CPL, gpw = 32 / L;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / L, sub = lane % L;
  const int slots = (kPoolThreads / 32) * gpw;
  const int64_t r0 = graph_ptr[g], r1 = graph_ptr[g + 1];
  const int c0 = sub * 8, stride = L * 8;
  if (grp < gpw) {
    float part[CPL][8] = {};
    for (int64_t row = r0 + warp * gpw + grp; row < r1; row += slots) {
      float x[CPL][8];
      load_chunks<DT, CPL>(h, row, c0, stride, x);
#pragma unroll
      for (int q = 0; q < CPL; ++q)
#pragma unroll
        for (int k = 0; k < 8; ++k) part[q][k] += x[q][k];
    }
    const int slot = warp * gpw + grp;
#pragma unroll
    for (int q = 0; q < CPL; ++q)
#pragma unroll
      for (int k = 0; k < 8; ++k) s_part[slot * width + c0 + q * stride + k] = part[q][k];
  }
  __syncthreads();
  const float inv_n = 1.0f / (float)(r1 - r0);
  for (int c = threadIdx.x; c < width; c += blockDim.x) {
    float t = 0.f;
    for (int q = 0; q < slots; ++q) t += s_part[q * width + c];
    act_store(u, g, c, t * inv_n);
  }
  for (int k = threadIdx.x; k < u.ld - width; k += blockDim.x) {
    float v = 0.f;
    if (k < kStaticWidth) {
      const double* fs_mean = norm + 6;
      const double* fs_std = norm + 11;
      v = (float)((fs_raw[g * kStaticWidth + k] - fs_mean[k]) / fs_std[k]);
    }
    act_store(u, g, width + k, v);
  }
}

// Second stage of the fused readout (see tc_gemm.cu pool_chunk): per graph, the block
// sums it owns in fixed block order, divided by N_g; then the static features.
__global__ void __launch_bounds__(128) k_pool_combine(const float* __restrict__ part, const float* __restrict__ whole,
                                                      const int* __restrict__ graph_ptr, int width,
                                                      const double* __restrict__ fs_raw, const double* __restrict__ norm,
                                                      ActView u) {
  pdl_begin();
  // one thread per 4 columns: the first block's partial and the following block sums of the
  // graph's 32-row blocks are loaded up to 16 float4 at a time (one L2 round trip per 16
  // blocks: a 300-node graph spans <= 11) and added in block order (fp64)
  const int g = blockIdx.x;
  const int gs = graph_ptr[g], ge = graph_ptr[g + 1];
  const int bf = gs >> 5, bl = (ge - 1) >> 5;
  const double inv_n = 1.0 / (double)(ge - gs);
  const int64_t rs = 2 * (int64_t)width;  // a block's two partial rows
  for (int c = threadIdx.x * 4; c < width; c += blockDim.x * 4) {
    double t[4];
    if (bf == bl) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(whole + (int64_t)g * width + c));
      t[0] = v.x; t[1] = v.y; t[2] = v.z; t[3] = v.w;
    } else {
      constexpr int kB = 16;
      float4 w[kB];
      // batch 0: the first block's partial row, then the middle blocks (slot 0) and the last block
      w[0] = __ldg(reinterpret_cast<const float4*>(part + ((int64_t)bf * 2 + ((gs & 31) == 0 ? 0 : 1)) * width + c));
#pragma unroll
      for (int j = 1; j < kB; ++j)
        if (bf + j <= bl) w[j] = __ldg(reinterpret_cast<const float4*>(part + (int64_t)(bf + j) * rs + c));
      t[0] = w[0].x; t[1] = w[0].y; t[2] = w[0].z; t[3] = w[0].w;
#pragma unroll
      for (int j = 1; j < kB; ++j)
        if (bf + j <= bl) {
          t[0] += w[j].x; t[1] += w[j].y; t[2] += w[j].z; t[3] += w[j].w;
        }
      for (int b = bf + kB; b <= bl; b += kB) {  // larger graphs: further batches, in order
#pragma unroll
        for (int j = 0; j < kB; ++j)
          if (b + j <= bl) w[j] = __ldg(reinterpret_cast<const float4*>(part + (int64_t)(b + j) * rs + c));
#pragma unroll
        for (int j = 0; j < kB; ++j)
          if (b + j <= bl) {
            t[0] += w[j].x; t[1] += w[j].y; t[2] += w[j].z; t[3] += w[j].w;
          }
      }
    }
    float o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) o[k] = (float)(t[k] * inv_n);
    if (u.dtype == DIPPM_DT_BF16) {
      __nv_bfloat162 h[2] = {__floats2bfloat162_rn(o[0], o[1]), __floats2bfloat162_rn(o[2], o[3])};
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(u.base) + (int64_t)g * u.ld + c) = *reinterpret_cast<uint2*>(h);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) act_store(u, g, c + k, o[k]);
    }
  }
  for (int k = threadIdx.x; k < u.ld - width; k += blockDim.x) {
    float v = 0.f;
    if (k < kStaticWidth) v = (float)((fs_raw[g * kStaticWidth + k] - norm[6 + k]) / norm[11 + k]);
    act_store(u, g, width + k, v);
  }
}

// MLP baseline input (gnn.py:253-255 with normalize_fs :96-97): u[g] = [(fs-mu)/sigma | 0].
__global__ void k_fs_normalize(const double* __restrict__ fs_raw, int64_t G, const double* __restrict__ norm,
                               ActView u, int cols) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= G * cols) return;
  const int64_t g = i / cols;
  const int c = (int)(i % cols);
  float v = 0.f;
  if (c < kStaticWidth) v = (float)((fs_raw[g * kStaticWidth + c] - norm[6 + c]) / norm[11 + c]);
  act_store(u, g, c, v);
}

// node -> graph id (for kernels that need g(v) per row).
__global__ void k_node_graph(const int* __restrict__ graph_ptr, int* __restrict__ node_graph) {
  const int g = blockIdx.x;
  for (int v = graph_ptr[g] + threadIdx.x; v < graph_ptr[g + 1]; v += blockDim.x) node_graph[v] = g;
}

}  // namespace dippm

using namespace dippm;

extern "C" {

// Rows per block chosen so the grid is a whole number of waves of resident blocks (the
// kernels are latency bound; a short last wave left ~30 % of the SMs idle, and the per-block
// CSR staging / barrier / fold tail is paid once per block): waves = ceil(N / (256 * P)) with
// P the resident blocks on the GPU, rows = ceil(N / (waves * P)) <= kRowsPerBlockT.
static int wave_rows_t(int64_t N, int blocks_per_sm) {
  const int64_t P = (int64_t)num_sms() * std::max(1, blocks_per_sm);
  const int64_t waves = std::max<int64_t>(1, (N + kRowsPerBlockT * P - 1) / (kRowsPerBlockT * P));
  return (int)std::max<int64_t>(1, (N + waves * P - 1) / (waves * P));
}
constexpr int kColsumBlocksPerSm = 4;  // upper bound of the agg^T kernels' residency (sizing only)

// Upper bound of the grid of a fused-bias agg^T launch with <= num_nodes rows (one partial
// row per block).  Without the fused reduction the kernels use 64-row blocks
// (dippm_colsum_blocks), so callers reducing the partials themselves see a fixed count.
static int64_t colsum_bound(int64_t num_nodes) {
  const int64_t P = (int64_t)num_sms() * kColsumBlocksPerSm;
  const int64_t waves = std::max<int64_t>(1, (num_nodes + kRowsPerBlock * P - 1) / (kRowsPerBlock * P));
  return std::max<int64_t>(ceil_div_i(num_nodes, kRowsPerBlock), waves * P);
}

// Deferred bias fold (the consumer -- the layer's weight-gradient GEMM -- folds the partial rows):
// the kernel stores its partial-row count as int32 in the last row of colsum_partial, a level-2
// row the deferred mode never uses.  dippm_gemm finds it the same way (dippm_colsum_count_slot).
static int32_t* deferred_count_slot(float* colsum_partial, int64_t N, int width) {
  const int64_t nb = colsum_bound(N);
  return reinterpret_cast<int32_t*>(colsum_partial + (nb + colsum_groups((int)nb) - 1) * (int64_t)width);
}
int32_t* dippm_colsum_count_slot(float* colsum_partial, int64_t num_nodes, int32_t width) {
  return deferred_count_slot(colsum_partial, num_nodes, width);
}

int32_t dippm_colsum_blocks(int64_t num_nodes) { return ceil_div_i(num_nodes, kRowsPerBlock); }
int32_t dippm_colsum_rows(int64_t num_nodes) {
  const int nblk = (int)colsum_bound(num_nodes);
  return nblk + colsum_groups(nblk);
}
int32_t dippm_colsum_sync_ints(int64_t num_nodes) { return colsum_groups((int)colsum_bound(num_nodes)) + 1; }

// 8-column chunks per lane: the lanes of a row (chunks / CPL) must tile a warp, so widths of
// 8 * 2^k chunks use CPL 1 / 2 / 4 and widths of 3 * 2^k chunks (24, 48, 96, 192, 384, 768
// columns) CPL 3
// dynamic shared memory launchable without the opt-in attribute: 48 KB less the kernels' static
// arrays (up to ~18 KB in k_aggregate_t)
constexpr size_t kDynSmemNoAttr = 24 * 1024;

static int cpl_for(int width) {
  const int chunks = width / 8;
  const int third = chunks / 3;
  if (chunks % 3 == 0 && third <= 32 && (third & (third - 1)) == 0) return 3;
  return chunks >= 128 ? 4 : (chunks >= 64 ? 2 : 1);
}

int32_t dippm_sage_aggregate(dippm_act_t h, dippm_act_t m_out, dippm_act_t self_out, int64_t N, int32_t width,
                             const int32_t* rowptr, const int32_t* col, const float* inv_deg, void* stream) {
  DIPPM_ARG_CHECK(N >= 1 && width >= 8 && width % 8 == 0, "sage_aggregate: width %d must be a multiple of 8", width);
  const int cpl = cpl_for(width);
  DIPPM_ARG_CHECK((width / 8) % cpl == 0 && (width / 8) / cpl <= 32 && 32 % ((width / 8) / cpl) == 0,
                  "sage_aggregate: unsupported width %d", width);
  DIPPM_ARG_CHECK(!self_out.data || self_out.dtype == m_out.dtype, "sage_aggregate: self_out dtype");
  cudaStream_t s = (cudaStream_t)stream;
  const int rpb = wave_rows_t(N, 4);
  const int grid = ceil_div_i(N, rpb);
  ActView hv = make_view(h), mv = make_view(m_out), sv = make_view(self_out);
#define DIPPM_AGG(DI, DO, C) \
  DIPPM_LAUNCH_PDL(k_aggregate<DI, DO, C>, dim3(grid), dim3(kAggThreads), 0, s, hv, mv, sv, N, rpb, width, rowptr, col, \
                   inv_deg)
#define DIPPM_AGG_C(DI, DO) \
  do { if (cpl == 4) DIPPM_AGG(DI, DO, 4); else if (cpl == 3) DIPPM_AGG(DI, DO, 3); else if (cpl == 2) DIPPM_AGG(DI, DO, 2); \
       else DIPPM_AGG(DI, DO, 1); } while (0)
#define DIPPM_AGG_O(DI)                                                   \
  do {                                                                    \
    if (m_out.dtype == DIPPM_DT_BF16) DIPPM_AGG_C(DI, DIPPM_DT_BF16);     \
    else if (m_out.dtype == DIPPM_DT_TF32X3) DIPPM_AGG_C(DI, DIPPM_DT_TF32X3); \
    else DIPPM_AGG_C(DI, DIPPM_DT_F32);                                   \
  } while (0)
  if (h.dtype == DIPPM_DT_BF16) DIPPM_AGG_O(DIPPM_DT_BF16);
  else if (h.dtype == DIPPM_DT_TF32X3) DIPPM_AGG_O(DIPPM_DT_TF32X3);
  else DIPPM_AGG_O(DIPPM_DT_F32);
#undef DIPPM_AGG_O
#undef DIPPM_AGG_C
#undef DIPPM_AGG
  DIPPM_LAUNCH_CHECK("k_aggregate");
  return DIPPM_OK;
}

static int launch_aggregate_t(dippm_act_t B, int32_t width, int64_t N, int32_t write_agg, const int32_t* t_rowptr,
                              const int32_t* t_col, const float* inv_deg, float* colsum_partial, ReadoutArgs ro,
                              bool readout, float* bias_out, int32_t* sync, cudaStream_t s) {
  DIPPM_ARG_CHECK(!bias_out || sync, "sage_aggregate_t: bias_grad needs the sync counters");
  DIPPM_ARG_CHECK(N >= 1 && width >= 8 && width % 8 == 0, "sage_aggregate_t: bad width %d", width);
  const int cpl = cpl_for(width);
  const int L = (width / 8) / cpl;
  DIPPM_ARG_CHECK((width / 8) % cpl == 0 && L <= 32 && 32 % L == 0, "sage_aggregate_t: unsupported width %d", width);
  size_t smem = (size_t)(kAggThreads / 32) * (32 / L) * width * sizeof(float);
  DIPPM_ARG_CHECK(smem <= 160 * 1024, "sage_aggregate_t: width %d too large", width);
  DIPPM_ARG_CHECK(!bias_out || width / 4 <= kAggThreads, "sage_aggregate_t: fused bias reduce needs width <= %d",
                  4 * kAggThreads);
  if (bias_out) smem = std::max(smem, (size_t)kAggThreads * 4 * sizeof(double));  // fold scratch
  // bias_out: fold in the kernel; sync only: deferred fold (wave-sized blocks, row count to the
  // slot); neither: caller-reduced partials over fixed 64-row blocks
  int rpb = (bias_out || sync) ? wave_rows_t(N, readout ? 2 : 3) : kRowsPerBlock;
  if (ceil_div_i(N, rpb) > colsum_bound(N)) rpb = kRowsPerBlock;           // partial rows are sized for this bound
  if (!bias_out && sync) sync = deferred_count_slot(colsum_partial, N, width);
  const int grid = ceil_div_i(N, rpb);
  ActView bv = make_view(B);
#define DIPPM_AGGT(D, C, R)                                                                                      \
  do {                                                                                                           \
    static bool attr_set = false; /* once per instantiation: dynamic + static can pass 48 KB */              \
    if (!attr_set && smem > kDynSmemNoAttr) {                                                                     \
      DIPPM_CUDA_CHECK(cudaFuncSetAttribute(k_aggregate_t<D, C, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));  \
      attr_set = true;                                                                                             \
    }                                                                                                             \
    DIPPM_LAUNCH_PDL(k_aggregate_t<D, C, R>, dim3(grid), dim3(kAggThreads), smem, s, bv, width, N, rpb, write_agg,     \
                     t_rowptr, t_col, inv_deg, colsum_partial, ro, bias_out, sync);                             \
  } while (0)
#define DIPPM_AGGT_C(D, R) \
  do { if (cpl == 4) DIPPM_AGGT(D, 4, R); else if (cpl == 3) DIPPM_AGGT(D, 3, R); else if (cpl == 2) DIPPM_AGGT(D, 2, R); \
       else DIPPM_AGGT(D, 1, R); } while (0)
#define DIPPM_AGGT_R(D) do { if (readout) DIPPM_AGGT_C(D, true); else DIPPM_AGGT_C(D, false); } while (0)
  if (B.dtype == DIPPM_DT_BF16) DIPPM_AGGT_R(DIPPM_DT_BF16);
  else if (B.dtype == DIPPM_DT_TF32X3) DIPPM_AGGT_R(DIPPM_DT_TF32X3);
  else DIPPM_AGGT_R(DIPPM_DT_F32);
#undef DIPPM_AGGT_R
#undef DIPPM_AGGT_C
#undef DIPPM_AGGT
  DIPPM_LAUNCH_CHECK("k_aggregate_t");
  return DIPPM_OK;
}

static int launch_readout_bits(dippm_act_t B, int32_t width, int64_t N, const int32_t* t_rowptr, const int32_t* t_col,
                               const float* inv_deg, float* colsum_partial, ReadoutArgs ro, float* bias_out,
                               int32_t* sync, cudaStream_t s) {
  DIPPM_ARG_CHECK(N >= 1 && width % 256 == 0 && width <= 1024, "readout_aggregate_t: width %d must be 256/512/768/1024",
                  width);
  DIPPM_ARG_CHECK(!bias_out || sync, "readout_aggregate_t: bias_grad needs the sync counters");
  int rpb = (bias_out || sync) ? wave_rows_t(N, width >= 768 ? 2 : 3) : kRowsPerBlock;  // the kernel's residency
  if (ceil_div_i(N, rpb) > colsum_bound(N)) rpb = kRowsPerBlock;
  if (!bias_out && sync) sync = deferred_count_slot(colsum_partial, N, width);  // deferred fold
  // [warp partials | fold scratch] then the staged bit words of rpb + halo rows
  const size_t smem = std::max((size_t)(kAggThreads / 32) * width * sizeof(float), (size_t)kAggThreads * 4 * sizeof(double)) +
                      (size_t)(width / 32) * (rpb + kBitsHalo) * sizeof(uint32_t);
  const int grid = ceil_div_i(N, rpb);
  static const bool generic = getenv("DIPPM_RO_GENERIC") != nullptr;  // A/B switch: the layout-generic kernel
  if (B.dtype == DIPPM_DT_BF16 && ro.bits_ld == 0 && B.ld % 8 == 0 && !generic) {
    __nv_bfloat16* bp = reinterpret_cast<__nv_bfloat16*>(B.data);
    if (bias_out || sync) {  // 4 resident blocks per SM at width <= 512
      rpb = wave_rows_t(N, width >= 768 ? 2 : 4);
      if (ceil_div_i(N, rpb) > colsum_bound(N)) rpb = kRowsPerBlock;
    }
    const int grid = ceil_div_i(N, rpb);
    const size_t smem = (size_t)(kAggThreads / 32) * width * sizeof(float) + (size_t)(width / 32) * (rpb + kBitsHalo) * 4;
#define DIPPM_RBM(C)                                                                                               \
  do {                                                                                                             \
    static bool attr_set = false;                                                                                  \
    if (!attr_set) {                                                                                               \
      DIPPM_CUDA_CHECK(cudaFuncSetAttribute(k_readout_bits_rm<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                                            160 * 1024));                                                          \
      attr_set = true;                                                                                             \
    }                                                                                                              \
    DIPPM_LAUNCH_PDL(k_readout_bits_rm<C>, dim3(grid), dim3(kAggThreads), smem, s, bp, B.ld, N, rpb, t_rowptr, t_col, \
                     inv_deg, colsum_partial, ro, bias_out, sync);                                                 \
  } while (0)
    if (width == 256) DIPPM_RBM(1);
    else if (width == 512) DIPPM_RBM(2);
    else if (width == 768) DIPPM_RBM(3);
    else DIPPM_RBM(4);
#undef DIPPM_RBM
    DIPPM_LAUNCH_CHECK("k_readout_bits_rm");
    return DIPPM_OK;
  }
  ActView bv = make_view(B);
#define DIPPM_RB(D, C)                                                                                            \
  do {                                                                                                            \
    static bool attr_set = false; /* dynamic + static shared memory can pass 48 KB at any size */               \
    if (!attr_set) {                                                                                              \
      DIPPM_CUDA_CHECK(cudaFuncSetAttribute(k_readout_agg_bits<D, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                            160 * 1024));                                                         \
      attr_set = true;                                                                                            \
    }                                                                                                             \
    DIPPM_LAUNCH_PDL(k_readout_agg_bits<D, C>, dim3(grid), dim3(kAggThreads), smem, s, bv, width, N, rpb, t_rowptr,   \
                     t_col, inv_deg, colsum_partial, ro, bias_out, sync);                                         \
  } while (0)
#define DIPPM_RB_C(D) \
  do { if (width == 256) DIPPM_RB(D, 1); else if (width == 512) DIPPM_RB(D, 2); else if (width == 768) DIPPM_RB(D, 3); else DIPPM_RB(D, 4); } while (0)
  if (B.dtype == DIPPM_DT_BF16) DIPPM_RB_C(DIPPM_DT_BF16);
  else if (B.dtype == DIPPM_DT_TF32X3) DIPPM_RB_C(DIPPM_DT_TF32X3);
  else DIPPM_RB_C(DIPPM_DT_F32);
#undef DIPPM_RB_C
#undef DIPPM_RB
  DIPPM_LAUNCH_CHECK("k_readout_agg_bits");
  return DIPPM_OK;
}

int32_t dippm_sage_aggregate_t(dippm_act_t B, int32_t width, int64_t N, int32_t write_agg, const int32_t* t_rowptr,
                               const int32_t* t_col, const float* inv_deg, float* colsum_partial, float* bias_grad,
                               int32_t* sync, void* stream) {
  ReadoutArgs ro{};
  return launch_aggregate_t(B, width, N, write_agg, t_rowptr, t_col, inv_deg, colsum_partial, ro, false, bias_grad,
                            sync, (cudaStream_t)stream);
}

int32_t dippm_readout_aggregate_t(const float* du, int64_t ld_du, const int32_t* graph_ptr, const int32_t* node_graph,
                                  dippm_act_t h3, dippm_act_t B, int32_t width, int64_t N, const int32_t* t_rowptr,
                                  const int32_t* t_col, const float* inv_deg, float* colsum_partial,
                                  float* bias_grad, int32_t* sync, const uint32_t* h3_bits, int64_t bits_ld,
                                  void* stream) {
  DIPPM_ARG_CHECK((h3_bits || h3.dtype == B.dtype) && ld_du % 4 == 0, "readout_aggregate_t: dtype / alignment");
  DIPPM_ARG_CHECK(!h3_bits || bits_ld >= N || bits_ld == 0, "readout_aggregate_t: bits_ld %lld < rows",
                  (long long)bits_ld);
  ReadoutArgs ro{du, ld_du, graph_ptr, node_graph, make_view(h3), h3_bits, bits_ld, (int64_t)(width >> 5)};
  if (h3_bits && width % 256 == 0 && width <= 1024)
    return launch_readout_bits(B, width, N, t_rowptr, t_col, inv_deg, colsum_partial, ro, bias_grad, sync,
                               (cudaStream_t)stream);
  return launch_aggregate_t(B, width, N, 1, t_rowptr, t_col, inv_deg, colsum_partial, ro, true, bias_grad, sync,
                            (cudaStream_t)stream);
}

int32_t dippm_readout_backward(const float* du, int64_t ld_du, const int32_t* graph_ptr, int64_t G, int32_t width,
                               dippm_act_t h3, dippm_act_t dz_out, int64_t N, void* stream) {
  DIPPM_ARG_CHECK(N >= 1 && G >= 1 && width % 8 == 0 && width / 8 <= kAggThreads, "readout_backward: bad args");
  k_readout_backward<<<dippm_colsum_blocks(N), kAggThreads, 0, (cudaStream_t)stream>>>(
      du, ld_du, width, make_view(h3), make_view(dz_out), N, graph_ptr, G);
  DIPPM_LAUNCH_CHECK("k_readout_backward");
  return DIPPM_OK;
}

int32_t dippm_reduce_rows(const float* in, int64_t rows, int64_t ld, int32_t cols, double scale, float* out,
                          void* stream) {
  DIPPM_ARG_CHECK(rows >= 0 && cols >= 1, "reduce_rows: bad shape");
  k_reduce_rows<<<ceil_div_i(cols, 32), 1024, 0, (cudaStream_t)stream>>>(in, rows, ld, cols, scale, out);
  DIPPM_LAUNCH_CHECK("k_reduce_rows");
  return DIPPM_OK;
}

int32_t dippm_pool_concat(dippm_act_t h, const int32_t* graph_ptr, int64_t G, int32_t width, const double* fs_raw,
                          const double* norm, dippm_act_t u, void* stream) {
  DIPPM_ARG_CHECK(G >= 1 && width >= 8 && width % 8 == 0 && u.ld >= width + 5, "pool_concat: bad args");
  const int cpl = cpl_for(width);
  const int L = (width / 8) / cpl;
  DIPPM_ARG_CHECK((width / 8) % cpl == 0 && L <= 32 && 32 % L == 0, "pool_concat: unsupported width %d", width);
  const size_t smem = (size_t)(kPoolThreads / 32) * (32 / L) * width * sizeof(float);
  DIPPM_ARG_CHECK(smem <= 160 * 1024, "pool_concat: width %d too large", width);
  cudaStream_t s = (cudaStream_t)stream;
  ActView hv = make_view(h), uv = make_view(u);
#define DIPPM_POOL(D, C)                                                                                         \
  do {                                                                                                           \
    static bool attr_set = false; /* once per instantiation: dynamic + static can pass 48 KB */              \
    if (!attr_set && smem > kDynSmemNoAttr) {                                                                     \
      DIPPM_CUDA_CHECK(cudaFuncSetAttribute(k_pool_concat<D, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));  \
      attr_set = true;                                                                                             \
    }                                                                                                             \
    k_pool_concat<D, C><<<(unsigned)G, kPoolThreads, smem, s>>>(hv, graph_ptr, width, fs_raw, norm, uv);         \
  } while (0)
#define DIPPM_POOL_C(D) \
  do { if (cpl == 4) DIPPM_POOL(D, 4); else if (cpl == 3) DIPPM_POOL(D, 3); else if (cpl == 2) DIPPM_POOL(D, 2); \
       else DIPPM_POOL(D, 1); } while (0)
  if (h.dtype == DIPPM_DT_BF16) DIPPM_POOL_C(DIPPM_DT_BF16);
  else if (h.dtype == DIPPM_DT_TF32X3) DIPPM_POOL_C(DIPPM_DT_TF32X3);
  else DIPPM_POOL_C(DIPPM_DT_F32);
#undef DIPPM_POOL_C
#undef DIPPM_POOL
  DIPPM_LAUNCH_CHECK("k_pool_concat");
  return DIPPM_OK;
}

int64_t dippm_pool_partial_rows(int64_t num_nodes) { return 2 * ((num_nodes + 31) / 32); }

int32_t dippm_pool_combine(const float* pool_partial, const float* pool_graph, const int32_t* graph_ptr, int64_t G,
                           int32_t width, const double* fs_raw, const double* norm, dippm_act_t u, void* stream) {
  DIPPM_ARG_CHECK(G >= 1 && width >= 4 && width % 4 == 0 && u.ld >= width + kStaticWidth && u.ld % 4 == 0,
                  "pool_combine: bad args");
  DIPPM_LAUNCH_PDL(k_pool_combine, dim3((unsigned)G), dim3(128), 0, (cudaStream_t)stream, pool_partial, pool_graph,
                   graph_ptr, width, fs_raw, norm, make_view(u));
  DIPPM_LAUNCH_CHECK("k_pool_combine");
  return DIPPM_OK;
}

int32_t dippm_fs_normalize(const double* fs_raw, int64_t G, const double* norm, dippm_act_t u, int32_t cols,
                           void* stream) {
  DIPPM_ARG_CHECK(G >= 1 && cols >= kStaticWidth && cols <= u.ld, "fs_normalize: bad shape");
  k_fs_normalize<<<ceil_div_i(G * cols, 256), 256, 0, (cudaStream_t)stream>>>(fs_raw, G, norm, make_view(u), cols);
  DIPPM_LAUNCH_CHECK("k_fs_normalize");
  return DIPPM_OK;
}

int32_t dippm_node_graph(const int32_t* graph_ptr, int64_t G, int32_t* node_graph, void* stream) {
  DIPPM_ARG_CHECK(G >= 1, "node_graph: no graphs");
  k_node_graph<<<(unsigned)G, 256, 0, (cudaStream_t)stream>>>(graph_ptr, node_graph);
  DIPPM_LAUNCH_CHECK("k_node_graph");
  return DIPPM_OK;
}

}  // extern "C"
