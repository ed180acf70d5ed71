// C-ABI plumbing: error state, device queries, MIG rule, Adam, weight packing.
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace dippm {

static thread_local char g_err[1024] = "";
static std::atomic<unsigned long long> g_launches{0};

void count_launches(int n) { g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* what) {
  set_error("CUDA error in %s: %s", what, cudaGetErrorString(e));
  return DIPPM_ERR_CUDA;
}

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n > 0 ? n : 148;
  }
  return cached[dev];
}

__global__ void k_mig_codes(const double* mem, int64_t stride, int64_t n, int8_t* codes, int32_t* nonfinite) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double a = mem[i * stride];
  if (!isfinite(a)) {
    atomicExch(nonfinite, 1);
    codes[i] = -1;
    return;
  }
  codes[i] = (int8_t)mig_rule(a);
}

struct PackSegs {
  int n;
  struct Seg {
    int64_t src_off, rows, cols, dst_col_off;
    ActView dst;
  } s[DIPPM_MAX_PACK_SEGS];
};

// numerics.py:93-114 in the same operation order (t already incremented; the two bias
// corrections are applied as multiplies by per-block reciprocals, fp64 throughout),
// fused with the refresh of the fp32 copy and of every GEMM operand copy.
__global__ void __launch_bounds__(256) k_adam_pack(double* __restrict__ p, double* __restrict__ m,
                                                   double* __restrict__ v, const float* __restrict__ g,
                                                   double gscale, int64_t n, double lr, double b1, double b2,
                                                   double eps, double bc1, double bc2, const int64_t* t_dev, int do_adam,
                                                   float* __restrict__ p32, PackSegs segs) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (t_dev && do_adam) {  // step count on the device (CUDA-graph replays): bias corrections from it
    __shared__ double s_bc[2];  // one pow pair per block, not per thread
    if (threadIdx.x == 0) {
      const double t = (double)t_dev[0];
      s_bc[0] = 1.0 - pow(b1, t);
      s_bc[1] = 1.0 - pow(b2, t);
    }
    __syncthreads();
    bc1 = s_bc[0];
    bc2 = s_bc[1];
  }
  const double inv_bc1 = 1.0 / bc1, inv_bc2 = 1.0 / bc2;
  for (; i < n; i += stride) {
    double val = p[i];
    if (do_adam) {
      double gi = (double)g[i] * gscale;
      double mi = m[i] * b1;
      mi += (1.0 - b1) * gi;
      double tmp = gi * gi;
      tmp *= 1.0 - b2;
      double vi = v[i] * b2;
      vi += tmp;
      double denom = vi * inv_bc2;  // v / (1 - b2^t) as a multiply by the per-block reciprocal
      denom = sqrt(denom);
      denom += eps;
      double step = mi * inv_bc1;
      step /= denom;
      step *= -lr;
      step += val;
      m[i] = mi;
      v[i] = vi;
      p[i] = step;
      val = step;
    }
    const float f = (float)val;
    p32[i] = f;
    for (int k = 0; k < segs.n; ++k) {
      const auto& sg = segs.s[k];
      const int64_t j = i - sg.src_off;
      if (j >= 0 && j < sg.rows * sg.cols) {  // 32-bit div/mod: segments are < 2^31 elements
        const uint32_t jj = (uint32_t)j, cc = (uint32_t)sg.cols;
        if ((cc & (cc - 1)) == 0) {  // power-of-two widths (the padded hidden sizes): shifts
          const int sh = __ffs(cc) - 1;
          act_store(sg.dst, jj >> sh, sg.dst_col_off + (jj & (cc - 1)), f);
        } else {
          act_store(sg.dst, jj / cc, sg.dst_col_off + jj % cc, f);
        }
      }
    }
  }
}

__global__ void k_step_counter(int64_t* t) { t[0] += 1; }

__global__ void k_pack(const double* __restrict__ w, int64_t rows, int64_t cols, int transpose, ActView dst) {
  // 32x32 tile transpose through shared memory when transpose != 0.
  __shared__ float tile[32][33];
  int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int64_t r = r0 + i, c = c0 + threadIdx.x;
    tile[i][threadIdx.x] = (r < rows && c < cols) ? (float)w[r * cols + c] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    if (transpose) {
      int64_t c = c0 + i, r = r0 + threadIdx.x;  // dst[c, r] = w[r, c]
      if (r < rows && c < cols) act_store(dst, c, r, tile[threadIdx.x][i]);
    } else {
      int64_t r = r0 + i, c = c0 + threadIdx.x;
      if (r < rows && c < cols) act_store(dst, r, c, tile[i][threadIdx.x]);
    }
  }
}

}  // namespace dippm

using namespace dippm;

extern "C" {

const char* dippm_last_error(void) { return g_err; }
int32_t dippm_abi_version(void) { return DIPPM_ABI_VERSION; }
uint64_t dippm_launch_count(void) { return g_launches.load(); }
int32_t dippm_device_sm_count(void) { return num_sms(); }

int32_t dippm_mig_code(double alpha_mb, int32_t* code) {
  if (!code) {
    set_error("dippm_mig_code: null output");
    return DIPPM_ERR_ARG;
  }
  if (!std::isfinite(alpha_mb)) {
    set_error("memory prediction is not finite: %g", alpha_mb);
    return DIPPM_ERR_NONFINITE;
  }
  *code = mig_rule(alpha_mb);
  return DIPPM_OK;
}

int32_t dippm_mig_codes(const double* mem_mb, int64_t stride, int64_t count, int8_t* codes, int32_t* nonfinite,
                        void* stream) {
  DIPPM_ARG_CHECK(count >= 0 && stride >= 1, "dippm_mig_codes: bad count/stride");
  if (count == 0) return DIPPM_OK;
  k_mig_codes<<<ceil_div_i(count, 256), 256, 0, (cudaStream_t)stream>>>(mem_mb, stride, count, codes, nonfinite);
  DIPPM_LAUNCH_CHECK("k_mig_codes");
  return DIPPM_OK;
}

int32_t dippm_adam_pack(double* params, double* m, double* v, const float* grads, double grad_scale, int64_t n,
                        int64_t t, const int64_t* t_dev, double lr, double beta1, double beta2, double eps,
                        int32_t do_adam, float* p32, const dippm_pack_seg_t* segs, int32_t nsegs, void* stream) {
  DIPPM_ARG_CHECK(n >= 0 && (t >= 1 || t_dev || !do_adam), "adam_pack: bad n/t");
  DIPPM_ARG_CHECK(nsegs >= 0 && nsegs <= DIPPM_MAX_PACK_SEGS, "adam_pack: %d segments (max %d)", nsegs,
                  DIPPM_MAX_PACK_SEGS);
  if (n == 0) return DIPPM_OK;
  PackSegs ps{};
  ps.n = nsegs;
  for (int k = 0; k < nsegs; ++k) {
    DIPPM_ARG_CHECK(segs[k].src_off >= 0 && segs[k].src_off + segs[k].rows * segs[k].cols <= n,
                    "adam_pack: segment %d out of range", k);
    ps.s[k].src_off = segs[k].src_off;
    ps.s[k].rows = segs[k].rows;
    ps.s[k].cols = segs[k].cols;
    ps.s[k].dst_col_off = segs[k].dst_col_off;
    ps.s[k].dst = make_view(segs[k].dst);
  }
  double bc1 = do_adam && t >= 1 ? 1.0 - pow(beta1, (double)t) : 1.0;
  double bc2 = do_adam && t >= 1 ? 1.0 - pow(beta2, (double)t) : 1.0;
  int blocks = (int)std::min<int64_t>(ceil_div_i(n, 256), 8 * num_sms());
  k_adam_pack<<<blocks, 256, 0, (cudaStream_t)stream>>>(params, m, v, grads, grad_scale, n, lr, beta1, beta2, eps,
                                                        bc1, bc2, t_dev, do_adam, p32, ps);
  DIPPM_LAUNCH_CHECK("k_adam_pack");
  return DIPPM_OK;
}

int32_t dippm_step_counter(int64_t* t_dev, void* stream) {
  k_step_counter<<<1, 1, 0, (cudaStream_t)stream>>>(t_dev);
  DIPPM_LAUNCH_CHECK("k_step_counter");
  return DIPPM_OK;
}

int32_t dippm_pack(const double* w, int64_t rows, int64_t cols, int32_t transpose, dippm_act_t dst, void* stream) {
  DIPPM_ARG_CHECK(rows > 0 && cols > 0, "dippm_pack: empty matrix");
  dim3 grid(ceil_div_i(cols, 32), ceil_div_i(rows, 32));
  k_pack<<<grid, dim3(32, 8), 0, (cudaStream_t)stream>>>(w, rows, cols, transpose, make_view(dst));
  DIPPM_LAUNCH_CHECK("k_pack");
  return DIPPM_OK;
}

}  // extern "C"
