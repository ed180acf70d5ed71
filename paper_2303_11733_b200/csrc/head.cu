// K5/K6 — FC head pieces that are not GEMMs, Huber loss, and the SIMT fp32
// GEMM backend (parity anchor for the tensor-core kernels, selected with
// backend = 1 in dippm_gemm).
//
// Head (gnn.py:265-284): a1 = u@W1+b1; x2 = relu(a1)*mask1; a2 = x2@W2+b2;
// x3 = relu(a2)*mask2; out = x3@W3+b3.  fc1/fc2 and their gradients run as
// tcgen05 GEMMs (dippm_gemm FWD / GATE / STORE / WGRAD); fc3 (3 outputs),
// its backward fused with the fc2 ReLU/dropout gate, the de-normalisation
// and the MIG pick run here.
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
  int kind;               // DIPPM_GEMM_*
  const float* bias;
  int relu;
  int drop_mode;
  float* mask;
  int64_t ldm;
  float p;
  uint64_t seed;
  ActView gate;
  float gate_scale;
  float* c;               // fp32 output (STORE / WGRAD)
  int64_t ldc;
  ActView out;            // FWD / GATE output view
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
      float v = acc[i][j];
      if (e.kind == DIPPM_GEMM_FWD) {
        if (e.bias) v += e.bias[n];
        if (e.relu) v = fmaxf(v, 0.f);
        if (e.drop_mode == 1) {
          v *= e.mask[m * e.ldm + n];
        } else if (e.drop_mode == 2) {
          float mk = uniform_hash(e.seed, (uint64_t)(m * e.ldm + n)) >= e.p ? 1.0f / (1.0f - e.p) : 0.f;
          e.mask[m * e.ldm + n] = mk;
          v *= mk;
        }
        act_store(e.out, m, n, v);
      } else if (e.kind == DIPPM_GEMM_GATE) {
        act_store(e.out, m, n, act_load(e.gate, m, n) > 0.f ? v * e.gate_scale : 0.f);
      } else {
        e.c[m * e.ldc + n] = v;
      }
    }
  }
}

// out[i*ldo + j] = scale * sum_s in[s*M*ldc + i*ldc + j] (fixed split order, fp64 sums)
__global__ void k_splitk_reduce(const float* __restrict__ in, int64_t splits, int64_t M, int64_t N, int64_t ldc,
                                double scale, float* __restrict__ out, int64_t ldo) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= M * N) return;
  const int64_t i = idx / N, j = idx % N;
  double a = 0.0;
  for (int64_t s = 0; s < splits; ++s) a += (double)in[s * M * ldc + i * ldc + j];
  out[i * ldo + j] = (float)(a * scale);
}

static int launch_simt(const Operand& A, const Operand& B, int64_t M, int64_t N, int64_t K, const Epi& e,
                       cudaStream_t s) {
  dim3 grid(ceil_div_i(N, kTN), ceil_div_i(M, kTM));
  k_simt_gemm<<<grid, 256, 0, s>>>(A, B, M, N, K, e);
  DIPPM_LAUNCH_CHECK("k_simt_gemm");
  return DIPPM_OK;
}

// ---------------------------------------------------------------------------
// fc3 (width -> 3) + de-normalisation (gnn.py:93-94) + MIG pick (mig.py:32-45):
// one warp per graph.
__global__ void k_fc3(ActView x3, int64_t G, int width, const float* __restrict__ w3, const float* __restrict__ b3,
                      float* __restrict__ out, const double* __restrict__ norm, double* __restrict__ y_pred,
                      int8_t* __restrict__ mig, int* nonfinite) {
  int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (g >= G) return;
  float s0 = 0.f, s1 = 0.f, s2 = 0.f;
  for (int j = lane; j < width; j += 32) {
    float x = act_load(x3, g, j);
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
      for (int k = 0; k < 3; ++k) y_pred[g * 3 + k] = (double)o3[k] * norm[3 + k] + norm[k];
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

// fc3 backward fused with the fc2 ReLU/dropout gate (gnn.py:293-298):
//   dW3[j,k] = sum_g x3[g,j] d3[g,k];  db3[k] = sum_g d3[g,k]
//   d2[g,j]  = (sum_k d3[g,k] W3[j,k]) * (x3[g,j] > 0 ? keep_scale : 0)
//   db2[j]   = sum_g d2[g,j]
// Block: 32 columns x 8 graph groups; fixed-order reductions (deterministic).
constexpr int kFc3Groups = 32;  // row groups per block (warps): 32 columns x 32 row groups
__global__ void __launch_bounds__(1024) k_fc3_backward(ActView x3, int64_t G, int width, const float* __restrict__ w3,
                                                      const float* __restrict__ d3, float keep_scale,
                                                      float* __restrict__ gw3, float* __restrict__ gb3, ActView d2,
                                                      float* __restrict__ gb2) {
  __shared__ float s[kFc3Groups][32][5];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + tx;
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, ab = 0.f;
  if (j < width) {
    const float w0 = w3[j * 3 + 0], w1 = w3[j * 3 + 1], w2 = w3[j * 3 + 2];
    int64_t g = ty;
    // 4 rows per step: all loads issued before the stores (d2 may alias nothing we read,
    // but the compiler cannot know), so each thread keeps 4 row loads in flight.
    for (; g + 3 * kFc3Groups < G; g += 4 * kFc3Groups) {
      float x[4], e[4][3];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        x[u] = act_load(x3, g + kFc3Groups * u, j);
        e[u][0] = __ldg(d3 + (g + kFc3Groups * u) * 3 + 0);
        e[u][1] = __ldg(d3 + (g + kFc3Groups * u) * 3 + 1);
        e[u][2] = __ldg(d3 + (g + kFc3Groups * u) * 3 + 2);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a0 = fmaf(x[u], e[u][0], a0);
        a1 = fmaf(x[u], e[u][1], a1);
        a2 = fmaf(x[u], e[u][2], a2);
        const float dx = e[u][0] * w0 + e[u][1] * w1 + e[u][2] * w2;
        const float dv = x[u] > 0.f ? dx * keep_scale : 0.f;
        act_store(d2, g + kFc3Groups * u, j, dv);
        ab += dv;
      }
    }
    for (; g < G; g += kFc3Groups) {
      const float x = act_load(x3, g, j);
      const float e0 = d3[g * 3 + 0], e1 = d3[g * 3 + 1], e2 = d3[g * 3 + 2];
      a0 = fmaf(x, e0, a0);
      a1 = fmaf(x, e1, a1);
      a2 = fmaf(x, e2, a2);
      const float dx = e0 * w0 + e1 * w1 + e2 * w2;
      const float dv = x > 0.f ? dx * keep_scale : 0.f;
      act_store(d2, g, j, dv);
      ab += dv;
    }
  }
  s[ty][tx][0] = a0;
  s[ty][tx][1] = a1;
  s[ty][tx][2] = a2;
  s[ty][tx][3] = ab;
  __syncthreads();
  if (ty == 0 && j < width) {
    float r0 = 0.f, r1 = 0.f, r2 = 0.f, rb = 0.f;
    for (int q = 0; q < kFc3Groups; ++q) {
      r0 += s[q][tx][0];
      r1 += s[q][tx][1];
      r2 += s[q][tx][2];
      rb += s[q][tx][3];
    }
    gw3[j * 3 + 0] = r0;
    gw3[j * 3 + 1] = r1;
    gw3[j * 3 + 2] = r2;
    gb2[j] = rb;
  }
  if (blockIdx.x == 0) {  // db3 = sum_g d3[g]: 1024 threads, fixed-order tree over thread partials
    __shared__ float sb[3][1024];
    float b0 = 0.f, b1 = 0.f, b2 = 0.f;
    for (int64_t g = threadIdx.x; g < G; g += blockDim.x) {
      b0 += d3[g * 3 + 0];
      b1 += d3[g * 3 + 1];
      b2 += d3[g * 3 + 2];
    }
    sb[0][threadIdx.x] = b0;
    sb[1][threadIdx.x] = b1;
    sb[2][threadIdx.x] = b2;
    __syncthreads();
    for (int w = 512; w > 0; w >>= 1) {
      if ((int)threadIdx.x < w)
        for (int k = 0; k < 3; ++k) sb[k][threadIdx.x] += sb[k][threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x < 3) gb3[threadIdx.x] = sb[threadIdx.x][0];
  }
}

// Column sums of an activation view [rows, cols] (fixed order): 32 columns x 8 row groups per block.
__global__ void __launch_bounds__(256) k_colsum_act(ActView a, int64_t rows, int cols, float* __restrict__ out) {
  __shared__ float s[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + tx;
  float acc = 0.f;
  if (c < cols) {
    int64_t r = ty;
    for (; r + 24 < rows; r += 32) {  // 4 independent loads in flight, summed in row order
      const float v0 = act_load(a, r, c), v1 = act_load(a, r + 8, c), v2 = act_load(a, r + 16, c),
                  v3 = act_load(a, r + 24, c);
      acc += v0;
      acc += v1;
      acc += v2;
      acc += v3;
    }
    for (; r < rows; r += 8) acc += act_load(a, r, c);
  }
  s[ty][tx] = acc;
  __syncthreads();
  if (ty == 0 && c < cols) {
    float t = 0.f;
    for (int q = 0; q < 8; ++q) t += s[q][tx];
    out[c] = t;
  }
}

// numerics.py:58-73 per graph, mean over the batch (gnn.py:402-404).
__global__ void k_huber(const float* __restrict__ out, const double* __restrict__ y_raw, int64_t G,
                        const double* __restrict__ norm, double delta, double grad_den, float* __restrict__ dout,
                        double* __restrict__ loss_out) {
  double l = 0.0, ape[3] = {0, 0, 0};
  for (int64_t g = threadIdx.x; g < G; g += blockDim.x) {
    double le = 0.0;
    for (int k = 0; k < 3; ++k) {
      double pred = (double)out[g * 3 + k];
      double y = y_raw[g * 3 + k];
      double t = (y - norm[k]) / norm[3 + k];
      double r = pred - t, a = fabs(r);
      bool quad = a <= delta;
      le += quad ? 0.5 * r * r : delta * (a - 0.5 * delta);
      double gr = quad ? r : delta * (r > 0 ? 1.0 : (r < 0 ? -1.0 : 0.0));
      if (dout) dout[g * 3 + k] = (float)(gr / 3.0 / grad_den);
      double den = pred * norm[3 + k] + norm[k];
      ape[k] += fabs(den - y) / fabs(y);
    }
    l += le / 3.0;
  }
  // fixed-order block sums (the fused head's loss unit runs the same reduction)
  __shared__ double s_w[8];
  const double tl = block_sum256(l, s_w);
  double ta[3];
  for (int k = 0; k < 3; ++k) ta[k] = block_sum256(ape[k], s_w);
  if (threadIdx.x == 0) {
    loss_out[0] = tl / (double)G;
    for (int k = 0; k < 3; ++k) loss_out[1 + k] = ta[k];
  }
}

}  // namespace dippm

using namespace dippm;

extern "C" {

int32_t dippm_fc3_forward(dippm_act_t x3, int64_t G, int32_t width, const float* w3, const float* b3, float* out_norm,
                          const double* norm, double* y_pred, int8_t* mig, int32_t* nonfinite, void* stream) {
  DIPPM_ARG_CHECK(G >= 1 && width >= 1, "fc3_forward: bad shape");
  DIPPM_ARG_CHECK(!y_pred || (mig && nonfinite && norm), "fc3_forward: y_pred needs norm, mig, nonfinite");
  k_fc3<<<ceil_div_i(G * 32, 256), 256, 0, (cudaStream_t)stream>>>(make_view(x3), G, width, w3, b3, out_norm, norm,
                                                                  y_pred, mig, nonfinite);
  DIPPM_LAUNCH_CHECK("k_fc3");
  return DIPPM_OK;
}

int32_t dippm_fc3_backward(dippm_act_t x3, int64_t G, int32_t width, const float* w3, const float* dout,
                           float keep_scale, float* grad_w3, float* grad_b3, dippm_act_t d2, float* grad_b2,
                           void* stream) {
  DIPPM_ARG_CHECK(G >= 1 && width >= 1, "fc3_backward: bad shape");
  k_fc3_backward<<<ceil_div_i(width, 32), 32 * kFc3Groups, 0, (cudaStream_t)stream>>>(make_view(x3), G, width, w3, dout,
                                                                          keep_scale, grad_w3, grad_b3,
                                                                          make_view(d2), grad_b2);
  DIPPM_LAUNCH_CHECK("k_fc3_backward");
  return DIPPM_OK;
}

int32_t dippm_colsum_act(dippm_act_t a, int64_t rows, int32_t cols, float* out, void* stream) {
  DIPPM_ARG_CHECK(rows >= 1 && cols >= 1, "colsum_act: bad shape");
  k_colsum_act<<<ceil_div_i(cols, 32), 256, 0, (cudaStream_t)stream>>>(make_view(a), rows, cols, out);
  DIPPM_LAUNCH_CHECK("k_colsum_act");
  return DIPPM_OK;
}

int32_t dippm_huber(const float* out_norm, const double* y_raw, int64_t G, const double* norm, double delta,
                    double grad_den, float* dout, double* loss_out, void* stream) {
  DIPPM_ARG_CHECK(G >= 1 && delta > 0, "huber: bad args");
  k_huber<<<1, 256, 0, (cudaStream_t)stream>>>(out_norm, y_raw, G, norm, delta, grad_den > 0 ? grad_den : (double)G,
                                               dout, loss_out);
  DIPPM_LAUNCH_CHECK("k_huber");
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
  Epi e{};
  e.kind = (int)a->kind;
  e.bias = a->bias;
  e.relu = (int)a->relu;
  e.drop_mode = (int)a->drop_mode;
  e.mask = a->mask;
  e.ldm = a->ldm;
  e.p = (float)a->drop_p;
  e.seed = a->seed;
  if (a->seed_dev) {  // host copy of the device counter is not available here: the SIMT anchor is eager-only
    int64_t t = 0;
    cudaMemcpyAsync(&t, a->seed_dev, sizeof(t), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    e.seed ^= (uint64_t)t * 0x9E3779B97F4A7C15ull;
  }
  e.gate = make_view(a->gate);
  e.gate_scale = (float)a->gate_scale;
  e.c = a->c;
  e.ldc = a->ldc;
  e.out = make_view(a->out);
  if (a->kind != DIPPM_GEMM_WGRAD) return launch_simt(A, B, a->M, a->N, a->K, e, s);
  // WGRAD: reduction over K split in `splits` contiguous chunks.
  int64_t splits = a->splits < 1 ? 1 : a->splits;
  const bool fused = a->tile_sync != nullptr;
  if (fused && !a->c) {  // no workspace (single split): compute into out, then scale in place
    DIPPM_ARG_CHECK(splits == 1 && a->out.data, "gemm WGRAD: fused reduce needs out and (splits > 1) c");
    e.c = reinterpret_cast<float*>(a->out.data);
    e.ldc = a->out.ld;
    int st = launch_simt(A, B, a->M, a->N, a->K, e, s);
    if (st) return st;
    k_splitk_reduce<<<ceil_div_i(a->M * a->N, 256), 256, 0, s>>>(e.c, 1, a->M, a->N, e.ldc, a->out_scale, e.c,
                                                                 e.ldc);
    DIPPM_LAUNCH_CHECK("k_splitk_reduce");
    return DIPPM_OK;
  }
  for (int64_t sp = 0; sp < splits; ++sp) {
    int64_t k0 = sp * a->K / splits, k1 = (sp + 1) * a->K / splits;
    Epi es = e;
    es.c = a->c + sp * a->M * a->ldc;
    if (k1 <= k0) {
      DIPPM_CUDA_CHECK(cudaMemsetAsync(es.c, 0, sizeof(float) * a->M * a->ldc, s));
      continue;
    }
    Operand As = A, Bs = B;
    As.p = (const char*)A.p + k0 * A.sc * (A.dtype == DIPPM_DT_BF16 ? 2 : 4);
    Bs.p = (const char*)B.p + k0 * B.sr * (B.dtype == DIPPM_DT_BF16 ? 2 : 4);
    int st = launch_simt(As, Bs, a->M, a->N, k1 - k0, es, s);
    if (st) return st;
  }
  if (fused) {
    DIPPM_ARG_CHECK(a->out.data != nullptr, "gemm WGRAD: fused reduce needs an out view");
    k_splitk_reduce<<<ceil_div_i(a->M * a->N, 256), 256, 0, s>>>(a->c, splits, a->M, a->N, a->ldc, a->out_scale,
                                                                 reinterpret_cast<float*>(a->out.data), a->out.ld);
    DIPPM_LAUNCH_CHECK("k_splitk_reduce");
  }
  return DIPPM_OK;
}

}  // extern "C"
