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
#include "common.cuh"

namespace dippm {

constexpr int kAggThreads = 256;
constexpr int kAggColCap = 2048;   // neighbour ids staged in shared memory per block
constexpr int kColsumRows = 64;    // rows per block for column partial sums

// Block handles a contiguous row range; lanes are grouped L per row
// (L = min(32, width/8)), each lane owning 8-column chunks.
__global__ void __launch_bounds__(kAggThreads) k_aggregate(ActView h, ActView m, ActView self_out, int64_t N,
                                                           int width, const int* __restrict__ rowptr,
                                                           const int* __restrict__ col,
                                                           const float* __restrict__ inv_deg, int rows_per_block) {
  __shared__ int s_col[kAggColCap];
  const int chunks = width >> 3;
  const int L = chunks >= 32 ? 32 : chunks;
  const int gpw = 32 / L;  // rows per warp per step
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / L, sub = lane % L;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = (N < r0 + rows_per_block) ? N : r0 + rows_per_block;
  if (r0 >= N) return;
  const int cbeg = rowptr[r0], cend = rowptr[r1];
  const bool staged = (cend - cbeg) <= kAggColCap;
  if (staged)
    for (int i = threadIdx.x; i < cend - cbeg; i += blockDim.x) s_col[i] = col[cbeg + i];
  __syncthreads();
  const int rows_per_step = (kAggThreads / 32) * gpw;
  for (int64_t row = r0 + warp * gpw + grp; row < r1; row += rows_per_step) {
    if (grp >= gpw) break;
    const int b = rowptr[row], e = rowptr[row + 1];
    const float w = inv_deg[row];
    for (int c = sub * 8; c < width; c += L * 8) {
      float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int j = b; j < e; ++j) {
        const int u = staged ? s_col[j - cbeg] : col[j];
        float x[8];
        act_load8(h, u, c, x);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] += x[k];
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] *= w;
      act_store8(m, row, c, acc);
      if (self_out.base) {
        float x[8];
        act_load8(h, row, c, x);
        act_store8(self_out, row, c, x);
      }
    }
  }
}

// Backward gather (mode 0) / readout backward (mode 1) with fused ReLU mask and
// per-block column partial sums of the produced dz (bias gradient).
template <int kMode>
__global__ void __launch_bounds__(kAggThreads) k_dz(const float* __restrict__ dA, int64_t ld_da, int width,
                                                     ActView gate, ActView dz, int64_t N,
                                                     const int* __restrict__ t_rowptr, const int* __restrict__ t_col,
                                                     const float* __restrict__ inv_deg,
                                                     const int* __restrict__ graph_ptr, int64_t G,
                                                     float* __restrict__ colsum_partial) {
  extern __shared__ float s_part[];  // [groups][width]
  const int chunks = width >> 3;
  const int groups = kAggThreads / chunks;  // >= 1 (width <= 2048)
  const int grp = threadIdx.x / chunks, ch = threadIdx.x % chunks;
  const int64_t r0 = (int64_t)blockIdx.x * kColsumRows;
  const int64_t r1 = (N < r0 + kColsumRows) ? N : r0 + kColsumRows;
  float part[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (grp < groups) {
    const int c = ch * 8;
    int g = 0;
    if (kMode == 1) {  // graph of the first row handled by this thread (binary search)
      int lo = 0, hi = (int)G;
      int64_t rr = r0 + grp;
      while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (graph_ptr[mid] <= rr) lo = mid; else hi = mid;
      }
      g = lo;
    }
    for (int64_t row = r0 + grp; row < r1; row += groups) {
      float v[8];
      if (kMode == 0) {
        const float4* p = reinterpret_cast<const float4*>(dA + row * ld_da + c);
        float4 a0 = p[0], a1 = p[1];
        v[0] = a0.x; v[1] = a0.y; v[2] = a0.z; v[3] = a0.w;
        v[4] = a1.x; v[5] = a1.y; v[6] = a1.z; v[7] = a1.w;
        const int b = t_rowptr[row], e = t_rowptr[row + 1];
        for (int j = b; j < e; ++j) {
          const int tv = t_col[j];
          const float w = inv_deg[tv];
          const float4* q = reinterpret_cast<const float4*>(dA + (int64_t)tv * ld_da + width + c);
          float4 b0 = q[0], b1 = q[1];
          v[0] += w * b0.x; v[1] += w * b0.y; v[2] += w * b0.z; v[3] += w * b0.w;
          v[4] += w * b1.x; v[5] += w * b1.y; v[6] += w * b1.z; v[7] += w * b1.w;
        }
      } else {
        while (graph_ptr[g + 1] <= row) ++g;
        const float inv_n = 1.0f / (float)(graph_ptr[g + 1] - graph_ptr[g]);
        const float* p = dA + (int64_t)g * ld_da + c;  // du rows (ld = width + 5) are not 16B aligned
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __ldg(p + k) * inv_n;
      }
      float hg[8];
      act_load8(gate, row, c, hg);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        v[k] = hg[k] > 0.f ? v[k] : 0.f;  // relu'(z) with z>0 <=> h>0 (gnn.py:227)
        part[k] += v[k];
      }
      act_store8(dz, row, c, v);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) s_part[grp * width + c + k] = part[k];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < width; c += blockDim.x) {
    float s = 0.f;
    for (int q = 0; q < groups; ++q) s += s_part[q * width + c];
    colsum_partial[(int64_t)blockIdx.x * width + c] = s;
  }
}

__global__ void k_reduce_rows(const float* __restrict__ in, int64_t rows, int64_t ld, int cols, double scale,
                              float* __restrict__ out) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  double s = 0.0;
  for (int64_t r = 0; r < rows; ++r) s += (double)in[r * ld + c];
  out[c] = (float)(s * scale);
}

// K4: one block per graph.
__global__ void __launch_bounds__(kAggThreads) k_pool_concat(ActView h, const int* __restrict__ graph_ptr,
                                                             int width, const float* __restrict__ fs_raw,
                                                             const double* __restrict__ norm,
                                                             float* __restrict__ u) {
  extern __shared__ float s_part[];
  const int g = blockIdx.x;
  const int chunks = width >> 3;
  const int groups = kAggThreads / chunks;
  const int grp = threadIdx.x / chunks, ch = threadIdx.x % chunks;
  const int64_t r0 = graph_ptr[g], r1 = graph_ptr[g + 1];
  const int ldu = width + kStaticWidth;
  if (grp < groups) {
    float part[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t row = r0 + grp; row < r1; row += groups) {
      float x[8];
      act_load8(h, row, ch * 8, x);
#pragma unroll
      for (int k = 0; k < 8; ++k) part[k] += x[k];
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) s_part[grp * width + ch * 8 + k] = part[k];
  }
  __syncthreads();
  const float inv_n = 1.0f / (float)(r1 - r0);
  for (int c = threadIdx.x; c < width; c += blockDim.x) {
    float s = 0.f;
    for (int q = 0; q < groups; ++q) s += s_part[q * width + c];
    u[(int64_t)g * ldu + c] = s * inv_n;
  }
  if (threadIdx.x < kStaticWidth) {
    const int k = threadIdx.x;
    const double* fs_mean = norm + 6;
    const double* fs_std = norm + 11;
    u[(int64_t)g * ldu + width + k] = (float)(((double)fs_raw[g * kStaticWidth + k] - fs_mean[k]) / fs_std[k]);
  }
}

}  // namespace dippm

using namespace dippm;

extern "C" {

int32_t dippm_colsum_blocks(int64_t num_nodes) { return ceil_div_i(num_nodes, kColsumRows); }

int32_t dippm_sage_aggregate(dippm_act_t h, dippm_act_t m_out, dippm_act_t self_out, int64_t N, int32_t width,
                             const int32_t* rowptr, const int32_t* col, const float* inv_deg, void* stream) {
  DIPPM_ARG_CHECK(N >= 1 && width >= 8 && width % 8 == 0, "sage_aggregate: width %d must be a multiple of 8", width);
  const int chunks = width / 8;
  const int L = chunks >= 32 ? 32 : chunks;
  const int gpw = 32 / L;
  const int rows_per_block = (kAggThreads / 32) * gpw * 4;
  k_aggregate<<<ceil_div_i(N, rows_per_block), kAggThreads, 0, (cudaStream_t)stream>>>(
      make_view(h), make_view(m_out), make_view(self_out), N, width, rowptr, col, inv_deg, rows_per_block);
  DIPPM_LAUNCH_CHECK("k_aggregate");
  return DIPPM_OK;
}

int32_t dippm_sage_backward_gather(const float* dA, int64_t ld_da, int32_t width, dippm_act_t h_prev,
                                   dippm_act_t dz_out, int64_t N, const int32_t* t_rowptr, const int32_t* t_col,
                                   const float* inv_deg, float* colsum_partial, void* stream) {
  DIPPM_ARG_CHECK(N >= 1 && width % 8 == 0 && width / 8 <= kAggThreads, "sage_backward_gather: bad width %d", width);
  const int groups = kAggThreads / (width / 8);
  size_t smem = (size_t)groups * width * sizeof(float);
  k_dz<0><<<dippm_colsum_blocks(N), kAggThreads, smem, (cudaStream_t)stream>>>(
      dA, ld_da, width, make_view(h_prev), make_view(dz_out), N, t_rowptr, t_col, inv_deg, nullptr, 0,
      colsum_partial);
  DIPPM_LAUNCH_CHECK("k_dz<gather>");
  return DIPPM_OK;
}

int32_t dippm_readout_backward(const float* du, int64_t ld_du, const int32_t* graph_ptr, int64_t G, int32_t width,
                               dippm_act_t h3, dippm_act_t dz_out, int64_t N, float* colsum_partial, void* stream) {
  DIPPM_ARG_CHECK(N >= 1 && G >= 1 && width % 8 == 0 && width / 8 <= kAggThreads, "readout_backward: bad args");
  const int groups = kAggThreads / (width / 8);
  size_t smem = (size_t)groups * width * sizeof(float);
  k_dz<1><<<dippm_colsum_blocks(N), kAggThreads, smem, (cudaStream_t)stream>>>(
      du, ld_du, width, make_view(h3), make_view(dz_out), N, nullptr, nullptr, nullptr, graph_ptr, G,
      colsum_partial);
  DIPPM_LAUNCH_CHECK("k_dz<readout>");
  return DIPPM_OK;
}

int32_t dippm_reduce_rows(const float* in, int64_t rows, int64_t ld, int32_t cols, double scale, float* out,
                          void* stream) {
  DIPPM_ARG_CHECK(rows >= 0 && cols >= 1, "reduce_rows: bad shape");
  k_reduce_rows<<<ceil_div_i(cols, 128), 128, 0, (cudaStream_t)stream>>>(in, rows, ld, cols, scale, out);
  DIPPM_LAUNCH_CHECK("k_reduce_rows");
  return DIPPM_OK;
}

int32_t dippm_pool_concat(dippm_act_t h, const int32_t* graph_ptr, int64_t G, int32_t width, const float* fs_raw,
                          const double* norm, float* u, void* stream) {
  DIPPM_ARG_CHECK(G >= 1 && width % 8 == 0 && width / 8 <= kAggThreads, "pool_concat: bad args");
  const int groups = kAggThreads / (width / 8);
  size_t smem = (size_t)groups * width * sizeof(float);
  k_pool_concat<<<(unsigned)G, kAggThreads, smem, (cudaStream_t)stream>>>(make_view(h), graph_ptr, width, fs_raw,
                                                                         norm, u);
  DIPPM_LAUNCH_CHECK("k_pool_concat");
  return DIPPM_OK;
}

}  // extern "C"
