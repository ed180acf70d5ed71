// MIG-pick parity for the bf16 predict path (mig.py:32-45).
//
// The bf16 forward's predicted memory is within the stated bf16 tolerance of the fp64
// reference, so its MIG pick can differ from the reference's only for graphs whose
// prediction lies within that band of a pick boundary (0 MB, the alpha <= 0 -> None rule,
// and the profile ceilings 5120/10240/20480/40960 MB).
// These kernels pick those graphs out of a batch, gather them into a compact sub-batch
// (node rows, edges re-based, static features) for an fp32 re-score, and scatter the
// fp32 predictions and picks back.  Batch layout: graph_ptr [G+1] (node rows), edge_ptr
// [G+1] (edges grouped by graph, global node ids).
#include "common.cuh"

namespace dippm {

constexpr int kSelThreads = 1024;

__device__ __forceinline__ bool near_ceiling(double mem, double band) {
  // the boundaries of mig_rule (common.cuh): alpha <= 0 -> None, then the four ceilings;
  // NaN compares false (NonFinite is flagged elsewhere)
  return fabs(mem) <= band || fabs(mem - 5120.0) <= band || fabs(mem - 10240.0) <= band || fabs(mem - 20480.0) <= band ||
         fabs(mem - 40960.0) <= band;
}

// One block: order-preserving compaction of the band graphs + exclusive prefix sums of
// their node and edge counts (totals[0] = count, [1] = nodes, [2] = edges).
__global__ void __launch_bounds__(kSelThreads) k_band_select(const double* __restrict__ y_pred, int64_t G,
                                                             double band, const int32_t* __restrict__ graph_ptr,
                                                             const int64_t* __restrict__ edge_ptr,
                                                             int32_t* __restrict__ sel_idx,
                                                             int32_t* __restrict__ sel_node_ptr,
                                                             int64_t* __restrict__ sel_edge_ptr,
                                                             int64_t* __restrict__ totals) {
  __shared__ int64_t s_warp[3][kSelThreads / 32];
  __shared__ int64_t s_base[3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_base[0] = s_base[1] = s_base[2] = 0;
  __syncthreads();
  for (int64_t g0 = 0; g0 < G; g0 += kSelThreads) {
    const int64_t g = g0 + threadIdx.x;
    int64_t v[3] = {0, 0, 0};
    if (g < G && near_ceiling(y_pred[g * 3 + 1], band)) {
      v[0] = 1;
      v[1] = graph_ptr[g + 1] - graph_ptr[g];
      v[2] = edge_ptr[g + 1] - edge_ptr[g];
    }
    int64_t incl[3] = {v[0], v[1], v[2]};
#pragma unroll
    for (int q = 0; q < 3; ++q) {
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t t = __shfl_up_sync(0xffffffffu, incl[q], o);
        if (lane >= o) incl[q] += t;
      }
      if (lane == 31) s_warp[q][warp] = incl[q];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        int64_t w = s_warp[q][lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int64_t t = __shfl_up_sync(0xffffffffu, w, o);
          if (lane >= o) w += t;
        }
        s_warp[q][lane] = w;  // inclusive over warps
      }
    }
    __syncthreads();
    int64_t excl[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) excl[q] = s_base[q] + (warp ? s_warp[q][warp - 1] : 0) + incl[q] - v[q];
    if (v[0]) {
      sel_idx[excl[0]] = (int32_t)g;
      sel_node_ptr[excl[0]] = (int32_t)excl[1];
      sel_edge_ptr[excl[0]] = excl[2];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
      for (int q = 0; q < 3; ++q) s_base[q] += s_warp[q][kSelThreads / 32 - 1];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    sel_node_ptr[s_base[0]] = (int32_t)s_base[1];
    sel_edge_ptr[s_base[0]] = s_base[2];
    totals[0] = s_base[0];
    totals[1] = s_base[1];
    totals[2] = s_base[2];
  }
}

// One CTA per selected graph: node rows (fp32 [n, 32]), edges re-based onto the sub-batch's
// node numbering, and the graph's static features.
__global__ void __launch_bounds__(256) k_gather_graphs(const int32_t* __restrict__ sel_idx,
                                                       const int32_t* __restrict__ sel_node_ptr,
                                                       const int64_t* __restrict__ sel_edge_ptr,
                                                       const int32_t* __restrict__ graph_ptr,
                                                       const int64_t* __restrict__ edge_ptr,
                                                       const float* __restrict__ x, const int64_t* __restrict__ src,
                                                       const int64_t* __restrict__ dst, const double* __restrict__ fs,
                                                       float* __restrict__ x_out, int64_t* __restrict__ src_out,
                                                       int64_t* __restrict__ dst_out, double* __restrict__ fs_out) {
  const int k = blockIdx.x;
  const int g = sel_idx[k];
  const int64_t n0 = graph_ptr[g], n = graph_ptr[g + 1] - n0, m0 = sel_node_ptr[k];
  const int64_t e0 = edge_ptr[g], ne = edge_ptr[g + 1] - e0, f0 = sel_edge_ptr[k];
  const float4* xs = reinterpret_cast<const float4*>(x + n0 * kFeatureWidth);
  float4* xd = reinterpret_cast<float4*>(x_out + m0 * kFeatureWidth);
  for (int64_t i = threadIdx.x; i < n * (kFeatureWidth / 4); i += blockDim.x) xd[i] = xs[i];
  const int64_t shift = m0 - n0;
  for (int64_t j = threadIdx.x; j < ne; j += blockDim.x) {
    src_out[f0 + j] = src[e0 + j] + shift;
    dst_out[f0 + j] = dst[e0 + j] + shift;
  }
  if (threadIdx.x < kStaticWidth) fs_out[k * kStaticWidth + threadIdx.x] = fs[(int64_t)g * kStaticWidth + threadIdx.x];
}

__global__ void k_scatter_rescore(const int32_t* __restrict__ sel_idx, int64_t count, const double* __restrict__ y_sub,
                                  const int8_t* __restrict__ mig_sub, double* __restrict__ y_pred,
                                  int8_t* __restrict__ mig) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= count) return;
  const int64_t g = sel_idx[k];
#pragma unroll
  for (int c = 0; c < 3; ++c) y_pred[g * 3 + c] = y_sub[k * 3 + c];
  mig[g] = mig_sub[k];
}

}  // namespace dippm

using namespace dippm;

extern "C" {

int32_t dippm_mig_band_select(const double* y_pred, int64_t num_graphs, double band_mb, const int32_t* graph_ptr,
                              const int64_t* edge_ptr, int32_t* sel_idx, int32_t* sel_node_ptr, int64_t* sel_edge_ptr,
                              int64_t* totals, void* stream) {
  DIPPM_ARG_CHECK(num_graphs >= 1 && y_pred && graph_ptr && edge_ptr && sel_idx && sel_node_ptr && sel_edge_ptr &&
                      totals, "mig_band_select: bad arguments");
  DIPPM_ARG_CHECK(band_mb >= 0.0, "mig_band_select: negative band");
  k_band_select<<<1, kSelThreads, 0, (cudaStream_t)stream>>>(y_pred, num_graphs, band_mb, graph_ptr, edge_ptr, sel_idx,
                                                             sel_node_ptr, sel_edge_ptr, totals);
  DIPPM_LAUNCH_CHECK("k_band_select");
  return DIPPM_OK;
}

int32_t dippm_gather_graphs(const int32_t* sel_idx, int64_t count, const int32_t* sel_node_ptr,
                            const int64_t* sel_edge_ptr, const int32_t* graph_ptr, const int64_t* edge_ptr,
                            const float* x, const int64_t* src, const int64_t* dst, const double* fs, float* x_out,
                            int64_t* src_out, int64_t* dst_out, double* fs_out, void* stream) {
  DIPPM_ARG_CHECK(count >= 0 && count < (1ll << 31), "gather_graphs: bad count");
  if (count == 0) return DIPPM_OK;
  k_gather_graphs<<<(unsigned)count, 256, 0, (cudaStream_t)stream>>>(sel_idx, sel_node_ptr, sel_edge_ptr, graph_ptr,
                                                                     edge_ptr, x, src, dst, fs, x_out, src_out,
                                                                     dst_out, fs_out);
  DIPPM_LAUNCH_CHECK("k_gather_graphs");
  return DIPPM_OK;
}

int32_t dippm_scatter_rescore(const int32_t* sel_idx, int64_t count, const double* y_sub, const int8_t* mig_sub,
                              double* y_pred, int8_t* mig, void* stream) {
  DIPPM_ARG_CHECK(count >= 0, "scatter_rescore: bad count");
  if (count == 0) return DIPPM_OK;
  k_scatter_rescore<<<ceil_div_i(count, 256), 256, 0, (cudaStream_t)stream>>>(sel_idx, count, y_sub, mig_sub, y_pred,
                                                                              mig);
  DIPPM_LAUNCH_CHECK("k_scatter_rescore");
  return DIPPM_OK;
}

}  // extern "C"
