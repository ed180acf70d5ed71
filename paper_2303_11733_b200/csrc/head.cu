// K5/K6 — FC head forward/backward, Huber loss, de-normalisation + MIG pick,
// and the SIMT fp32 GEMM that carries the head (M = #graphs, tiny next to the
// SAGE GEMMs: ~0.2% of the FLOPs) and serves as the parity anchor backend for
// the tensor-core kernels.
//
// Head (gnn.py:265-284): a1 = u@W1+b1; x2 = relu(a1)*mask1; a2 = x2@W2+b2;
// x3 = relu(a2)*mask2; out = x3@W3+b3.  Backward gnn.py:287-299.
#include <cmath>

#include "common.cuh"

namespace dippm {

// ---------------------------------------------------------------------------
// SIMT GEMM with general strides:  C(m,n) = epi( sum_k A(m,k) * B(k,n) ).
struct Operand {
  const void* p;
  int64_t sr, sc;        // element strides for (row, col) of the logical operand
  int64_t plane;         // tf32x3 lo plane offset
  int dtype;
};

__device__ __forceinline__ float op_load(const Operand& o, int64_t r, int64_t c) {
  int64_t off = r * o.sr + c * o.sc;
  if (o.dtype == DIPPM_DT_BF16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(o.p)[off]);
  const float* f = reinterpret_cast<const float*>(o.p);
  if (o.dtype == DIPPM_DT_TF32X3) return f[off] + f[off + o.plane];
  return f[off];
}

struct Epi {
  float alpha;
  const float* bias;      // [N]
  float* pre;             // store pre-activation (ld = ldc)
  int relu;
  const float* mask;      // multiply by mask(m,n) (ld = ldc)
  int mask_gen;           // generate inverted-dropout mask into `mask_out`
  float* mask_out;
  float p;
  uint64_t seed;
  const float* gate;      // zero where gate(m,n) <= 0 (ld = ldc)
  float* c;               // fp32 output
  int64_t ldc;
  ActView out;            // alternative output view (when c == nullptr)
};

constexpr int kTM = 64, kTN = 64, kTK = 16;

__global__ void __launch_bounds__(256) k_simt_gemm(Operand A, Operand B, int64_t M, int64_t N, int64_t K, Epi e) {
  __shared__ float sA[kTK][kTM + 4];
  __shared__ float sB[kTK][kTN + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t m0 = (int64_t)blockIdx.y * kTM, n0 = (int64_t)blockIdx.x * kTN;
  float acc[4][4] = {};
  for (int64_t k0 = 0; k0 < K; k0 += kTK) {
    for (int i = threadIdx.x; i < kTK * kTM; i += 256) {
      int kk = i / kTM, mm = i % kTM;
      int64_t m = m0 + mm, k = k0 + kk;
      sA[kk][mm] = (m < M && k < K) ? op_load(A, m, k) : 0.f;
    }
    for (int i = threadIdx.x; i < kTK * kTN; i += 256) {
      int kk = i / kTN, nn = i % kTN;
      int64_t n = n0 + nn, k = k0 + kk;
      sB[kk][nn] = (n < N && k < K) ? op_load(B, k, n) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kTK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sA[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = sB[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t n = n0 + tx * 4 + j;
      if (n >= N) continue;
      float v = acc[i][j] * e.alpha;
      if (e.bias) v += e.bias[n];
      int64_t idx = m * e.ldc + n;
      if (e.pre) e.pre[idx] = v;
      if (e.relu) v = fmaxf(v, 0.f);
      if (e.mask_gen) {
        float mk = (uniform_hash(e.seed, (uint64_t)idx) >= e.p) ? 1.0f / (1.0f - e.p) : 0.f;
        e.mask_out[idx] = mk;
        v *= mk;
      } else if (e.mask) {
        v *= e.mask[idx];
      }
      if (e.gate) v = e.gate[idx] > 0.f ? v : 0.f;
      if (e.c) e.c[idx] = v;
      else act_store(e.out, m, n, v);
    }
  }
}

static int launch_simt(const Operand& A, const Operand& B, int64_t M, int64_t N, int64_t K, const Epi& e,
                       cudaStream_t s) {
  dim3 grid(ceil_div_i(N, kTN), ceil_div_i(M, kTM));
  k_simt_gemm<<<grid, 256, 0, s>>>(A, B, M, N, K, e);
  DIPPM_LAUNCH_CHECK("k_simt_gemm");
  return DIPPM_OK;
}

static Epi epi_plain(float* c, int64_t ldc) {
  Epi e{};
  e.alpha = 1.f;
  e.c = c;
  e.ldc = ldc;
  return e;
}

static Operand dense(const float* p, int64_t sr, int64_t sc) {
  Operand o{p, sr, sc, 0, DIPPM_DT_F32};
  return o;
}

// fc3 (width -> 3) + optional de-normalisation and MIG pick: one warp per graph.
__global__ void k_fc3(const float* __restrict__ x3, int64_t G, int width, const float* __restrict__ w3,
                      const float* __restrict__ b3, float* __restrict__ out, const double* __restrict__ norm,
                      double* __restrict__ y_pred, int8_t* __restrict__ mig, int* nonfinite) {
  int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (g >= G) return;
  float s0 = 0.f, s1 = 0.f, s2 = 0.f;
  for (int j = lane; j < width; j += 32) {
    float x = x3[g * width + j];
    s0 = fmaf(x, w3[j * 3 + 0], s0);
    s1 = fmaf(x, w3[j * 3 + 1], s1);
    s2 = fmaf(x, w3[j * 3 + 2], s2);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  if (lane == 0) {
    float o3[3] = {s0 + b3[0], s1 + b3[1], s2 + b3[2]};
    for (int k = 0; k < 3; ++k) out[g * 3 + k] = o3[k];
    if (y_pred) {
      for (int k = 0; k < 3; ++k) y_pred[g * 3 + k] = (double)o3[k] * norm[3 + k] + norm[k];  // gnn.py:93-94
      double mem = y_pred[g * 3 + 1];
      if (!isfinite(mem)) {
        atomicExch(nonfinite, 1);
        mig[g] = -1;
      } else {
        mig[g] = (int8_t)mig_rule(mem);
      }
    }
  }
}

// numerics.py:58-73 per graph, mean over the batch (gnn.py:402-404).
__global__ void k_huber(const float* __restrict__ out, const float* __restrict__ y_raw, int64_t G,
                        const double* __restrict__ norm, double delta, float* __restrict__ dout,
                        double* __restrict__ loss_out) {
  __shared__ double s_loss[256], s_ape[3][256];
  double l = 0.0, ape[3] = {0, 0, 0};
  for (int64_t g = threadIdx.x; g < G; g += blockDim.x) {
    double le = 0.0;
    for (int k = 0; k < 3; ++k) {
      double pred = (double)out[g * 3 + k];
      double y = (double)y_raw[g * 3 + k];
      double t = (y - norm[k]) / norm[3 + k];
      double r = pred - t, a = fabs(r);
      bool quad = a <= delta;
      le += quad ? 0.5 * r * r : delta * (a - 0.5 * delta);
      double gr = quad ? r : delta * (r > 0 ? 1.0 : (r < 0 ? -1.0 : 0.0));
      dout[g * 3 + k] = (float)(gr / 3.0 / (double)G);
      double den = pred * norm[3 + k] + norm[k];
      ape[k] += fabs(den - y) / fabs(y);
    }
    l += le / 3.0;
  }
  s_loss[threadIdx.x] = l;
  for (int k = 0; k < 3; ++k) s_ape[k][threadIdx.x] = ape[k];
  __syncthreads();
  if (threadIdx.x == 0) {
    double tl = 0, ta[3] = {0, 0, 0};
    for (int i = 0; i < blockDim.x; ++i) {
      tl += s_loss[i];
      for (int k = 0; k < 3; ++k) ta[k] += s_ape[k][i];
    }
    loss_out[0] = tl / (double)G;
    for (int k = 0; k < 3; ++k) loss_out[1 + k] = ta[k];
  }
}

__global__ void k_colsum(const float* __restrict__ d, int64_t rows, int cols, float* __restrict__ out) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  float s = 0.f;
  for (int64_t r = 0; r < rows; ++r) s += d[r * cols + c];
  out[c] = s;
}

struct HeadOffsets {
  int64_t w1, b1, w2, b2, w3, b3, total;
};
static HeadOffsets head_offsets(int width) {
  HeadOffsets o;
  int64_t in1 = width + kStaticWidth;
  o.w1 = 0;
  o.b1 = o.w1 + in1 * width;
  o.w2 = o.b1 + width;
  o.b2 = o.w2 + (int64_t)width * width;
  o.w3 = o.b2 + width;
  o.b3 = o.w3 + (int64_t)width * 3;
  o.total = o.b3 + 3;
  return o;
}

}  // namespace dippm

using namespace dippm;

extern "C" {

int32_t dippm_head_forward(const float* u, int64_t G, int32_t width, const float* head_w, float* cache, float* masks,
                           int32_t mask_mode, float dropout_p, uint64_t seed, float* out_norm, const double* norm,
                           double* y_pred, int8_t* mig, int32_t* nonfinite, void* stream) {
  DIPPM_ARG_CHECK(G >= 1 && width >= 1, "head_forward: bad shape");
  DIPPM_ARG_CHECK(mask_mode >= 0 && mask_mode <= 2, "head_forward: bad mask_mode");
  DIPPM_ARG_CHECK(mask_mode == 0 || masks, "head_forward: masks buffer required in train mode");
  cudaStream_t s = (cudaStream_t)stream;
  HeadOffsets o = head_offsets(width);
  const int64_t in1 = width + kStaticWidth;
  const int64_t GW = G * width;
  float *a1 = cache, *x2 = cache + GW, *a2 = cache + 2 * GW, *x3 = cache + 3 * GW;
  for (int layer = 0; layer < 2; ++layer) {
    const float* x = layer == 0 ? u : x2;
    int64_t K = layer == 0 ? in1 : width;
    Epi e = epi_plain(layer == 0 ? x2 : x3, width);
    e.bias = head_w + (layer == 0 ? o.b1 : o.b2);
    e.pre = layer == 0 ? a1 : a2;
    e.relu = 1;
    float* mk = masks ? masks + layer * GW : nullptr;
    if (mask_mode == 1) e.mask = mk;
    if (mask_mode == 2) {
      e.mask_gen = 1;
      e.mask_out = mk;
      e.p = dropout_p;
      e.seed = seed * 2 + layer;
    }
    int st = launch_simt(dense(x, K, 1), dense(head_w + (layer == 0 ? o.w1 : o.w2), width, 1), G, width, K, e, s);
    if (st) return st;
  }
  k_fc3<<<ceil_div_i(G * 32, 256), 256, 0, s>>>(x3, G, width, head_w + o.w3, head_w + o.b3, out_norm, norm, y_pred,
                                              mig, nonfinite);
  DIPPM_LAUNCH_CHECK("k_fc3");
  return DIPPM_OK;
}

int32_t dippm_huber(const float* out_norm, const float* y_raw, int64_t G, const double* norm, double delta,
                    float* dout, double* loss_out, void* stream) {
  DIPPM_ARG_CHECK(G >= 1 && delta > 0, "huber: bad args");
  k_huber<<<1, 256, 0, (cudaStream_t)stream>>>(out_norm, y_raw, G, norm, delta, dout, loss_out);
  DIPPM_LAUNCH_CHECK("k_huber");
  return DIPPM_OK;
}

size_t dippm_head_scratch_floats(int64_t G, int32_t width) { return (size_t)(2 * G * width); }

int32_t dippm_head_backward(const float* u, int64_t G, int32_t width, const float* head_w, const float* cache,
                            const float* masks, int32_t use_masks, const float* dout, float* grads_head, float* du,
                            float* scratch, void* stream) {
  DIPPM_ARG_CHECK(G >= 1 && width >= 1, "head_backward: bad shape");
  cudaStream_t s = (cudaStream_t)stream;
  HeadOffsets o = head_offsets(width);
  const int64_t in1 = width + kStaticWidth;
  const int64_t GW = G * width;
  const float *a1 = cache, *x2 = cache + GW, *a2 = cache + 2 * GW, *x3 = cache + 3 * GW;
  float* d2 = scratch;       // [G, width]
  float* d1 = scratch + GW;  // [G, width]
  int st;
  // fc3: dW3 = x3^T d3, db3 = sum d3, then d2 = (d3 @ W3^T) * mask2 * (a2 > 0)
  st = launch_simt(dense(x3, 1, width), dense(dout, 3, 1), width, 3, G, epi_plain(grads_head + o.w3, 3), s);
  if (st) return st;
  k_colsum<<<1, 32, 0, s>>>(dout, G, 3, grads_head + o.b3);
  {
    Epi e = epi_plain(d2, width);
    if (use_masks) e.mask = masks + GW;
    e.gate = a2;
    st = launch_simt(dense(dout, 3, 1), dense(head_w + o.w3, 1, 3), G, width, 3, e, s);
    if (st) return st;
  }
  // fc2
  st = launch_simt(dense(x2, 1, width), dense(d2, width, 1), width, width, G, epi_plain(grads_head + o.w2, width), s);
  if (st) return st;
  k_colsum<<<ceil_div_i(width, 128), 128, 0, s>>>(d2, G, width, grads_head + o.b2);
  {
    Epi e = epi_plain(d1, width);
    if (use_masks) e.mask = masks;
    e.gate = a1;
    st = launch_simt(dense(d2, width, 1), dense(head_w + o.w2, 1, width), G, width, width, e, s);
    if (st) return st;
  }
  // fc1
  st = launch_simt(dense(u, 1, in1), dense(d1, width, 1), in1, width, G, epi_plain(grads_head + o.w1, width), s);
  if (st) return st;
  k_colsum<<<ceil_div_i(width, 128), 128, 0, s>>>(d1, G, width, grads_head + o.b1);
  st = launch_simt(dense(d1, width, 1), dense(head_w + o.w1, 1, width), G, in1, width, epi_plain(du, in1), s);
  if (st) return st;
  DIPPM_LAUNCH_CHECK_N(3, "head_backward");
  return DIPPM_OK;
}

// SIMT backend of dippm_gemm (parity anchor for the tensor-core kernels).
int32_t dippm_gemm_simt_impl(const dippm_gemm_args_t* a, cudaStream_t s) {
  auto operand = [](const dippm_act_t& v, int mn_major, bool is_b) {
    Operand o;
    o.p = v.data;
    o.plane = v.plane_stride;
    o.dtype = (int)v.dtype;
    // Logical A is (m, k); logical B is (k, n).
    // K-major storage: A[m*ld + k], B stored as [n, k] -> B(k,n) = p[n*ld + k].
    // MN-major storage: A stored [k, m] -> A(m,k) = p[k*ld + m]; B stored [k, n].
    if (!is_b) {
      o.sr = mn_major ? 1 : v.ld;
      o.sc = mn_major ? v.ld : 1;
    } else {
      o.sr = mn_major ? v.ld : 1;
      o.sc = mn_major ? 1 : v.ld;
    }
    return o;
  };
  Operand A = operand(a->a, (int)a->a_mn_major, false);
  Operand B = operand(a->b, (int)a->b_mn_major, true);
  if (a->kind == DIPPM_GEMM_FWD) {
    Epi e{};
    e.alpha = 1.f;
    e.bias = a->bias;
    e.relu = (int)a->relu;
    e.out = make_view(a->out);
    return launch_simt(A, B, a->M, a->N, a->K, e, s);
  }
  if (a->kind == DIPPM_GEMM_STORE) return launch_simt(A, B, a->M, a->N, a->K, epi_plain(a->c, a->ldc), s);
  // WGRAD: reduction over K split in `splits` chunks of whole 64-row blocks.
  int64_t splits = a->splits < 1 ? 1 : a->splits;
  int64_t kb = ceil_div_i(a->K, 64);
  int64_t per = (kb + splits - 1) / splits;
  for (int64_t sp = 0; sp < splits; ++sp) {
    int64_t k0 = sp * per * 64, k1 = std::min<int64_t>(a->K, (sp + 1) * per * 64);
    float* c = a->c + sp * a->M * a->ldc;
    if (k1 <= k0) {
      DIPPM_CUDA_CHECK(cudaMemsetAsync(c, 0, sizeof(float) * a->M * a->ldc, s));
      continue;
    }
    Operand As = A, Bs = B;
    As.p = (const char*)A.p + k0 * A.sc * (A.dtype == DIPPM_DT_BF16 ? 2 : 4);
    Bs.p = (const char*)B.p + k0 * B.sr * (B.dtype == DIPPM_DT_BF16 ? 2 : 4);
    int st = launch_simt(As, Bs, a->M, a->N, k1 - k0, epi_plain(c, a->ldc), s);
    if (st) return st;
  }
  return DIPPM_OK;
}

}  // extern "C"
