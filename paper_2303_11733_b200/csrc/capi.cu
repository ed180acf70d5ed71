// C-ABI plumbing: error state, device queries, MIG rule, Adam, weight packing.
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>

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

bool pdl_enabled() {
  static const bool on = [] {
    // measured: no gain inside the captured step (724 vs 730 us), so off unless DIPPM_PDL=1
    const char* e = getenv("DIPPM_PDL");
    return e && e[0] == '1';
  }();
  return on;
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

// Vectorised variant: 4 consecutive parameters per thread (16/32-byte loads and stores),
// the packing of GEMM operand copies specialised on their dtype.  Valid when every
// segment's src_off and cols are multiples of 4 (the padded layout guarantees it); the
// arithmetic per element is exactly k_adam_pack's.
template <int DT>
__global__ void __launch_bounds__(256) k_adam_pack4(double* __restrict__ p, double* __restrict__ m,
                                                    double* __restrict__ v, const float* __restrict__ g,
                                                    double gscale, int64_t n, double lr, double b1, double b2,
                                                    double eps, double bc1, double bc2, const int64_t* t_dev,
                                                    int do_adam, float* __restrict__ p32, PackSegs segs) {
  pdl_begin();
  const int64_t n4 = n >> 2;
  // warm this thread's first group in L1 while thread 0 evaluates the bias corrections
  const int64_t q0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q0 < n4) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p + (q0 << 2)));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(g + (q0 << 2)));
    if (do_adam) {
      asm volatile("prefetch.global.L1 [%0];" ::"l"(m + (q0 << 2)));
      asm volatile("prefetch.global.L1 [%0];" ::"l"(v + (q0 << 2)));
    }
  }
  if (t_dev && do_adam) {
    // the two fp64 pows (long dependent chains) run in two warps at once; the grid is one wave
    // (the launcher), so every block pays this latency once, concurrently
    __shared__ double s_bc[2];
    if ((threadIdx.x & 31) == 0 && threadIdx.x < 64) {
      const double t = (double)t_dev[0];
      s_bc[threadIdx.x >> 5] = 1.0 - pow(threadIdx.x ? b2 : b1, t);
    }
    __syncthreads();
    bc1 = s_bc[0];
    bc2 = s_bc[1];
  }
  const double inv_bc1 = 1.0 / bc1, inv_bc2 = 1.0 / bc2;
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {  // the < 4 trailing parameters (no packing segments there)
    const int64_t i = (n4 << 2) + threadIdx.x;
    double val = p[i];
    if (do_adam) {
      const double gi = (double)g[i] * gscale;
      double mi = m[i] * b1;
      mi += (1.0 - b1) * gi;
      double tmp = gi * gi;
      tmp *= 1.0 - b2;
      double vi = v[i] * b2;
      vi += tmp;
      double denom = vi * inv_bc2;
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
    p32[i] = (float)val;
  }
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n4; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q << 2;
    double val[4];
    {
      const double2 a = reinterpret_cast<const double2*>(p + i)[0], b = reinterpret_cast<const double2*>(p + i)[1];
      val[0] = a.x; val[1] = a.y; val[2] = b.x; val[3] = b.y;
    }
    if (do_adam) {
      const float4 g4 = reinterpret_cast<const float4*>(g + i)[0];
      const double2 ma = reinterpret_cast<const double2*>(m + i)[0], mb = reinterpret_cast<const double2*>(m + i)[1];
      const double2 va = reinterpret_cast<const double2*>(v + i)[0], vb = reinterpret_cast<const double2*>(v + i)[1];
      const double gg[4] = {(double)g4.x * gscale, (double)g4.y * gscale, (double)g4.z * gscale, (double)g4.w * gscale};
      const double mm[4] = {ma.x, ma.y, mb.x, mb.y}, vv[4] = {va.x, va.y, vb.x, vb.y};
      double mo[4], vo[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        double mi = mm[k] * b1;
        mi += (1.0 - b1) * gg[k];
        double tmp = gg[k] * gg[k];
        tmp *= 1.0 - b2;
        double vi = vv[k] * b2;
        vi += tmp;
        double denom = vi * inv_bc2;
        denom = sqrt(denom);
        denom += eps;
        double step = mi * inv_bc1;
        step /= denom;
        step *= -lr;
        step += val[k];
        mo[k] = mi;
        vo[k] = vi;
        val[k] = step;
      }
      reinterpret_cast<double2*>(m + i)[0] = make_double2(mo[0], mo[1]);
      reinterpret_cast<double2*>(m + i)[1] = make_double2(mo[2], mo[3]);
      reinterpret_cast<double2*>(v + i)[0] = make_double2(vo[0], vo[1]);
      reinterpret_cast<double2*>(v + i)[1] = make_double2(vo[2], vo[3]);
      reinterpret_cast<double2*>(p + i)[0] = make_double2(val[0], val[1]);
      reinterpret_cast<double2*>(p + i)[1] = make_double2(val[2], val[3]);
    }
    const float f[4] = {(float)val[0], (float)val[1], (float)val[2], (float)val[3]};
    reinterpret_cast<float4*>(p32 + i)[0] = make_float4(f[0], f[1], f[2], f[3]);
    for (int k = 0; k < segs.n; ++k) {
      const auto& sg = segs.s[k];
      const int64_t j = i - sg.src_off;
      if ((uint64_t)j >= (uint64_t)(sg.rows * sg.cols)) continue;
      // segments hold one weight matrix (< 2^31 elements): 32-bit index arithmetic
      const uint32_t j32 = (uint32_t)j, cols = (uint32_t)sg.cols;
      const int64_t r = j32 / cols, c = sg.dst_col_off + j32 % cols;
      if constexpr (DT == DIPPM_DT_BF16) {
        __nv_bfloat162 h[2] = {__floats2bfloat162_rn(f[0], f[1]), __floats2bfloat162_rn(f[2], f[3])};
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(sg.dst.base) + r * sg.dst.ld + c) =
            *reinterpret_cast<uint2*>(h);
      } else if constexpr (DT == DIPPM_DT_TF32X3) {
        float hi[4], lo[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          hi[e] = tf32_hi(f[e]);
          lo[e] = tf32_rn(f[e] - hi[e]);
        }
        float* d = reinterpret_cast<float*>(sg.dst.base) + r * sg.dst.ld + c;
        *reinterpret_cast<float4*>(d) = make_float4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<float4*>(d + sg.dst.plane_stride) = make_float4(lo[0], lo[1], lo[2], lo[3]);
      } else {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(sg.dst.base) + r * sg.dst.ld + c) =
            make_float4(f[0], f[1], f[2], f[3]);
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
  // vectorised path: 4 parameters per thread when every segment is 4-aligned and all
  // operand copies share one dtype; the <4 tail (and any other layout) runs the scalar kernel
  bool vec = true;
  for (int k = 0; k < nsegs; ++k)
    vec &= segs[k].src_off % 4 == 0 && segs[k].cols % 4 == 0 && segs[k].dst_col_off % 4 == 0 &&
           segs[k].dst.ld % 4 == 0 && segs[k].dst.plane_stride % 4 == 0 && (uintptr_t)segs[k].dst.data % 16 == 0 &&
           segs[k].src_off + segs[k].rows * segs[k].cols <= (n & ~int64_t(3)) && segs[k].dst.dtype == segs[0].dst.dtype;
  vec &= ((uintptr_t)params | (uintptr_t)m | (uintptr_t)v | (uintptr_t)grads | (uintptr_t)p32) % 32 == 0;
  const int64_t n4 = vec ? (n & ~int64_t(3)) : 0;
  if (n4) {
    const int b4 = (int)std::min<int64_t>(ceil_div_i(n4 / 4, 256), 3 * num_sms());  // one wave (76 regs: 3 / SM)
    const int dt = nsegs ? (int)segs[0].dst.dtype : DIPPM_DT_F32;
    if (dt == DIPPM_DT_BF16)
      DIPPM_LAUNCH_PDL(k_adam_pack4<DIPPM_DT_BF16>, dim3(b4), dim3(256), 0, (cudaStream_t)stream, params, m, v, grads, grad_scale, n, lr, beta1,
                                                                      beta2, eps, bc1, bc2, t_dev, do_adam, p32, ps);
    else if (dt == DIPPM_DT_TF32X3)
      DIPPM_LAUNCH_PDL(k_adam_pack4<DIPPM_DT_TF32X3>, dim3(b4), dim3(256), 0, (cudaStream_t)stream, params, m, v, grads, grad_scale, n, lr,
                                                                        beta1, beta2, eps, bc1, bc2, t_dev, do_adam,
                                                                        p32, ps);
    else
      DIPPM_LAUNCH_PDL(k_adam_pack4<DIPPM_DT_F32>, dim3(b4), dim3(256), 0, (cudaStream_t)stream, params, m, v, grads, grad_scale, n, lr, beta1,
                                                                     beta2, eps, bc1, bc2, t_dev, do_adam, p32, ps);
    DIPPM_LAUNCH_CHECK("k_adam_pack4");
    return DIPPM_OK;
  }
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
