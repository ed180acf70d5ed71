// fp64 scalar numerics of the drop-in `numerics` module (reference numerics.py:23-114).
//
// These are the per-record building blocks the reference's training loop calls
// (huber_loss, adam_step) plus its small dense helpers (matmul, add, scale, relu).
// Every operation is written with explicit round-to-nearest intrinsics so nvcc
// cannot contract a multiply and an add into an FMA: the element-wise results
// are then bit-identical to numpy's (IEEE mul/add/div/sqrt, same operation
// order), and the Huber mean uses numpy's pairwise summation order
// (numpy/_core/src/umath/loops_utils.h.src, DOUBLE_pairwise_sum), so
// huber_loss and adam_step reproduce the reference bit for bit.  matmul is a
// plain fp64 tiled GEMM (OpenBLAS's summation order is not reproducible; the
// reference's own tests hold it to 1e-10).
#include <cmath>

#include "common.cuh"

namespace dippm {

// numpy's pairwise sum (blocks of 128, 8 accumulators inside a block, sequential below 8).
__device__ double pairwise_sum(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise_sum(a, n2), pairwise_sum(a + n2, n - n2));
}

// numerics.py:58-73: r = pred - target; 0.5 r^2 (|r| <= delta) else delta (|r| - 0.5 delta);
// grad = (r or delta sign r) / size.
__global__ void k_huber_f64_elems(const double* __restrict__ pred, const double* __restrict__ target, int64_t n,
                                  double delta, double* __restrict__ grad, double* __restrict__ elems) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double r = __dadd_rn(pred[i], -target[i]);
  const double a = fabs(r);
  const bool quad = a <= delta;
  const double lin = __dmul_rn(delta, __dadd_rn(a, -__dmul_rn(0.5, delta)));
  elems[i] = quad ? __dmul_rn(__dmul_rn(0.5, r), r) : lin;
  const double sgn = r > 0.0 ? 1.0 : (r < 0.0 ? -1.0 : (r == 0.0 ? 0.0 : r));  // np.sign (NaN stays NaN)
  grad[i] = __ddiv_rn(quad ? r : __dmul_rn(delta, sgn), (double)n);
}

__global__ void k_mean_pairwise(const double* __restrict__ elems, int64_t n, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = __ddiv_rn(pairwise_sum(elems, n), (double)n);
}

// numerics.py:93-114 statement by statement (bc1 = 1 - beta1**t, bc2 = 1 - beta2**t and the
// scalar factors c1 = 1 - beta1, c2 = 1 - beta2 come from the host, where Python computes them).
__global__ void k_adam_f64(const double* __restrict__ param, const double* __restrict__ grad,
                           double* __restrict__ m, double* __restrict__ v, double* __restrict__ out, int64_t n,
                           double neg_lr, double b1, double b2, double c1, double c2, double eps, double bc1,
                           double bc2) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double g = grad[i];
  double mi = __dmul_rn(m[i], b1);              // state.m *= beta1
  mi = __dadd_rn(mi, __dmul_rn(c1, g));         // state.m += (1 - beta1) * grad
  double tmp = __dmul_rn(g, g);                 // tmp = grad * grad
  tmp = __dmul_rn(tmp, c2);                     // tmp *= 1 - beta2
  double vi = __dmul_rn(v[i], b2);              // state.v *= beta2
  vi = __dadd_rn(vi, tmp);                      // state.v += tmp
  double denom = __ddiv_rn(vi, bc2);            // v / (1 - beta2**t)
  denom = __dsqrt_rn(denom);
  denom = __dadd_rn(denom, eps);
  double step = __ddiv_rn(mi, bc1);             // m / (1 - beta1**t)
  step = __ddiv_rn(step, denom);
  step = __dmul_rn(step, neg_lr);               // step *= -lr
  step = __dadd_rn(step, param[i]);             // step += param
  m[i] = mi;
  v[i] = vi;
  out[i] = step;
}

// numerics.py:23-42: add, scale, relu (np.maximum(a, 0.0): NaN propagates, -0.0 stays).
__global__ void k_ew_f64(int op, const double* __restrict__ a, const double* __restrict__ b, double s,
                         double* __restrict__ out, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = a[i];
  if (op == 0) out[i] = __dadd_rn(x, b[i]);
  else if (op == 1) out[i] = __dmul_rn(x, s);
  else out[i] = (x >= 0.0 || x != x) ? x : 0.0;
}

// numerics.py:23-28 (matmul): fp64 C[M,N] = A[M,K] B[K,N], 32x32 tiles staged in shared memory.
__global__ void __launch_bounds__(256) k_dgemm(const double* __restrict__ A, const double* __restrict__ B,
                                               double* __restrict__ Cm, int64_t M, int64_t K, int64_t N) {
  __shared__ double sa[32][33], sb[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads, 4 rows each
  const int64_t row0 = blockIdx.y * 32, col = blockIdx.x * 32 + tx;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t k0 = 0; k0 < K; k0 += 32) {
    for (int rr = ty; rr < 32; rr += 8) {
      const int64_t r = row0 + rr, k = k0 + tx;
      sa[rr][tx] = (r < M && k < K) ? A[r * K + k] : 0.0;
      const int64_t kb = k0 + rr;
      sb[rr][tx] = (kb < K && col < N) ? B[kb * N + col] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < 32; ++k) {
      const double bv = sb[k][tx];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = fma(sa[ty + 8 * q][k], bv, acc[q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t r = row0 + ty + 8 * q;
    if (r < M && col < N) Cm[r * N + col] = acc[q];
  }
}

}  // namespace dippm

using namespace dippm;

extern "C" {

int32_t dippm_huber_f64(const double* pred, const double* target, int64_t n, double delta, double* grad,
                        double* elems, double* loss, void* stream) {
  DIPPM_ARG_CHECK(n >= 1 && pred && target && grad && elems && loss, "huber_f64: bad arguments (n=%lld)",
                  (long long)n);
  DIPPM_ARG_CHECK(delta > 0.0, "huber_f64: delta must be positive");
  cudaStream_t s = (cudaStream_t)stream;
  k_huber_f64_elems<<<ceil_div_i(n, 256), 256, 0, s>>>(pred, target, n, delta, grad, elems);
  DIPPM_LAUNCH_CHECK("k_huber_f64_elems");
  k_mean_pairwise<<<1, 32, 0, s>>>(elems, n, loss);
  DIPPM_LAUNCH_CHECK("k_mean_pairwise");
  return DIPPM_OK;
}

int32_t dippm_adam(const double* param, const double* grad, double* m, double* v, double* param_out, int64_t n,
                   double lr, double beta1, double beta2, double eps, double one_minus_beta1,
                   double one_minus_beta2, double bias_corr1, double bias_corr2, void* stream) {
  DIPPM_ARG_CHECK(n >= 0 && (n == 0 || (param && grad && m && v && param_out)), "adam: bad arguments");
  if (n == 0) return DIPPM_OK;
  k_adam_f64<<<ceil_div_i(n, 256), 256, 0, (cudaStream_t)stream>>>(
      param, grad, m, v, param_out, n, -lr, beta1, beta2, one_minus_beta1, one_minus_beta2, eps, bias_corr1,
      bias_corr2);
  DIPPM_LAUNCH_CHECK("k_adam_f64");
  return DIPPM_OK;
}

int32_t dippm_elementwise_f64(int32_t op, const double* a, const double* b, double s, double* out, int64_t n,
                              void* stream) {
  DIPPM_ARG_CHECK(op >= 0 && op <= 2, "elementwise_f64: unknown op %d", op);
  DIPPM_ARG_CHECK(n >= 0 && (n == 0 || (a && out && (op != 0 || b))), "elementwise_f64: bad arguments");
  if (n == 0) return DIPPM_OK;
  k_ew_f64<<<ceil_div_i(n, 256), 256, 0, (cudaStream_t)stream>>>(op, a, b, s, out, n);
  DIPPM_LAUNCH_CHECK("k_ew_f64");
  return DIPPM_OK;
}

int32_t dippm_dgemm(const double* a, const double* b, double* c, int64_t M, int64_t K, int64_t N, void* stream) {
  DIPPM_ARG_CHECK(M >= 0 && K >= 0 && N >= 0, "dgemm: negative size");
  if (M == 0 || N == 0) return DIPPM_OK;
  DIPPM_ARG_CHECK(a && b && c, "dgemm: null operand");
  DIPPM_ARG_CHECK(M / 32 < 65535, "dgemm: M=%lld too large", (long long)M);
  dim3 grid(ceil_div_i(N, 32), ceil_div_i(M, 32));
  k_dgemm<<<grid, 256, 0, (cudaStream_t)stream>>>(a, b, c, M, K, N);
  DIPPM_LAUNCH_CHECK("k_dgemm");
  return DIPPM_OK;
}

}  // extern "C"
