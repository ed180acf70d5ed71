// Shared device helpers for the DIPPM B200 kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <utility>

#include "../../include/dippm_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "dippm_b200 targets sm_100a only"
#endif

namespace dippm {

constexpr int kFeatureWidth = 32;   // featurize.py:38
constexpr int kStaticWidth = 5;     // featurize.py:39
constexpr int kOutputs = 3;         // (latency_ms, memory_mb, energy_j), dataset.py:54-62

// Error plumbing (capi.cu owns the storage).
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);
#define DIPPM_CUDA_CHECK(expr)                                     \
  do {                                                             \
    cudaError_t _e = (expr);                                       \
    if (_e != cudaSuccess) return ::dippm::cuda_status(_e, #expr); \
  } while (0)
// Every kernel launch is counted (dippm_launch_count) so the bench can report
// exactly how many of this library's kernels ran in its timed region.
void count_launches(int n);
#define DIPPM_LAUNCH_CHECK_N(n, what)                              \
  do {                                                             \
    ::dippm::count_launches(n);                                    \
    cudaError_t _e = cudaGetLastError();                           \
    if (_e != cudaSuccess) return ::dippm::cuda_status(_e, what);  \
  } while (0)
#define DIPPM_LAUNCH_CHECK(what) DIPPM_LAUNCH_CHECK_N(1, what)
#define DIPPM_ARG_CHECK(cond, ...)                                 \
  do {                                                             \
    if (!(cond)) {                                                 \
      ::dippm::set_error(__VA_ARGS__);                             \
      return DIPPM_ERR_ARG;                                        \
    }                                                              \
  } while (0)

inline int ceil_div_i(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }
int num_sms();

// Programmatic dependent launch: the training step's kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization when DIPPM_PDL=1 (off by default: it measured no
// gain inside the captured CUDA-graph step), so a kernel's
// launch and prologue overlap its predecessor's tail.  Every such kernel calls pdl_begin() in
// every CTA before it touches memory the predecessor wrote (griddepcontrol.wait returns once the
// predecessor grid has completed and its writes are visible; it is a no-op without the
// attribute), then allows its own dependents to launch (they wait the same way).
__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
#define DIPPM_LAUNCH_PDL(...)                                       \
  do {                                                             \
    cudaError_t _le = ::dippm::launch_pdl(__VA_ARGS__);            \
    if (_le != cudaSuccess) return ::dippm::cuda_status(_le, "launch"); \
  } while (0)

// ---------------------------------------------------------------------------
// Activation storage.  A "plane pair" holds an fp32 value v as two fp32 planes
// (hi = tf32(v), lo = tf32(v - hi), both round-to-nearest) so the tensor
// cores' tf32 path can run the 3-pass split (hi*hi + hi*lo + lo*hi) at fp32
// accuracy.  bf16 mode stores one bf16 plane.

// Round-to-nearest tf32 (cvt.rna): |v - hi| <= 2^-11 |v|; lo = rna(v - hi) is
// itself exactly representable in tf32, so the tensor core reads both planes
// without further rounding and each 3-pass product carries ~2^-22 relative error.
__device__ __forceinline__ float tf32_rn(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}
__device__ __forceinline__ float tf32_hi(float v) { return tf32_rn(v); }

struct ActView {
  // Element (r, c) of plane p lives at base + p*plane_stride + r*ld + c.
  void* base;
  int64_t ld;            // elements
  int64_t plane_stride;  // elements (tf32x3 only)
  int dtype;             // DIPPM_DT_BF16 / DIPPM_DT_TF32X3 / DIPPM_DT_F32
};

__device__ __forceinline__ float act_load(const ActView& a, int64_t r, int64_t c) {
  if (a.dtype == DIPPM_DT_BF16) {
    return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(a.base)[r * a.ld + c]);
  } else if (a.dtype == DIPPM_DT_TF32X3) {
    const float* p = reinterpret_cast<const float*>(a.base) + r * a.ld + c;
    return p[0] + p[a.plane_stride];
  }
  return reinterpret_cast<const float*>(a.base)[r * a.ld + c];
}

__device__ __forceinline__ void act_store(const ActView& a, int64_t r, int64_t c, float v) {
  if (a.dtype == DIPPM_DT_BF16) {
    reinterpret_cast<__nv_bfloat16*>(a.base)[r * a.ld + c] = __float2bfloat16_rn(v);
  } else if (a.dtype == DIPPM_DT_TF32X3) {
    float* p = reinterpret_cast<float*>(a.base) + r * a.ld + c;
    float hi = tf32_hi(v);
    p[0] = hi;
    p[a.plane_stride] = tf32_rn(v - hi);
  } else {
    reinterpret_cast<float*>(a.base)[r * a.ld + c] = v;
  }
}

// 8 consecutive elements (c must be a multiple of 8 and rows 16B aligned).
__device__ __forceinline__ void act_load8(const ActView& a, int64_t r, int64_t c, float (&v)[8]) {
  if (a.dtype == DIPPM_DT_BF16) {
    const uint4 q = __ldg(reinterpret_cast<const uint4*>(
        reinterpret_cast<const __nv_bfloat16*>(a.base) + r * a.ld + c));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __bfloat1622float2(h[i]);
      v[2 * i] = f.x;
      v[2 * i + 1] = f.y;
    }
  } else {
    const float* p = reinterpret_cast<const float*>(a.base) + r * a.ld + c;
    float4 x0 = __ldg(reinterpret_cast<const float4*>(p));
    float4 x1 = __ldg(reinterpret_cast<const float4*>(p + 4));
    v[0] = x0.x; v[1] = x0.y; v[2] = x0.z; v[3] = x0.w;
    v[4] = x1.x; v[5] = x1.y; v[6] = x1.z; v[7] = x1.w;
    if (a.dtype == DIPPM_DT_TF32X3) {
      float4 y0 = __ldg(reinterpret_cast<const float4*>(p + a.plane_stride));
      float4 y1 = __ldg(reinterpret_cast<const float4*>(p + a.plane_stride + 4));
      v[0] += y0.x; v[1] += y0.y; v[2] += y0.z; v[3] += y0.w;
      v[4] += y1.x; v[5] += y1.y; v[6] += y1.z; v[7] += y1.w;
    }
  }
}

__device__ __forceinline__ void act_store8(const ActView& a, int64_t r, int64_t c, const float (&v)[8]) {
  if (a.dtype == DIPPM_DT_BF16) {
    uint4 q;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.base) + r * a.ld + c) = q;
  } else if (a.dtype == DIPPM_DT_TF32X3) {
    float* p = reinterpret_cast<float*>(a.base) + r * a.ld + c;
    float hi[8], lo[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      hi[i] = tf32_hi(v[i]);
      lo[i] = tf32_rn(v[i] - hi[i]);
    }
    reinterpret_cast<float4*>(p)[0] = make_float4(hi[0], hi[1], hi[2], hi[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(hi[4], hi[5], hi[6], hi[7]);
    reinterpret_cast<float4*>(p + a.plane_stride)[0] = make_float4(lo[0], lo[1], lo[2], lo[3]);
    reinterpret_cast<float4*>(p + a.plane_stride)[1] = make_float4(lo[4], lo[5], lo[6], lo[7]);
  } else {
    float* p = reinterpret_cast<float*>(a.base) + r * a.ld + c;
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
}

// Compile-time-dtype variants (memory-bound kernels specialise on the dtype so
// the loads/stores carry no runtime branches and fewer live registers).
template <int DT>
__device__ __forceinline__ void act_load8_t(const ActView& a, int64_t r, int64_t c, float (&v)[8]) {
  if constexpr (DT == DIPPM_DT_BF16) {
    const uint4 q = __ldg(reinterpret_cast<const uint4*>(
        reinterpret_cast<const __nv_bfloat16*>(a.base) + r * a.ld + c));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      v[2 * i] = f.x;
      v[2 * i + 1] = f.y;
    }
  } else {
    const float* p = reinterpret_cast<const float*>(a.base) + r * a.ld + c;
    const float4 x0 = __ldg(reinterpret_cast<const float4*>(p));
    const float4 x1 = __ldg(reinterpret_cast<const float4*>(p + 4));
    v[0] = x0.x; v[1] = x0.y; v[2] = x0.z; v[3] = x0.w;
    v[4] = x1.x; v[5] = x1.y; v[6] = x1.z; v[7] = x1.w;
    if constexpr (DT == DIPPM_DT_TF32X3) {
      const float4 y0 = __ldg(reinterpret_cast<const float4*>(p + a.plane_stride));
      const float4 y1 = __ldg(reinterpret_cast<const float4*>(p + a.plane_stride + 4));
      v[0] += y0.x; v[1] += y0.y; v[2] += y0.z; v[3] += y0.w;
      v[4] += y1.x; v[5] += y1.y; v[6] += y1.z; v[7] += y1.w;
    }
  }
}

template <int DT>
__device__ __forceinline__ void act_store8_t(const ActView& a, int64_t r, int64_t c, const float (&v)[8]) {
  if constexpr (DT == DIPPM_DT_BF16) {
    uint4 q;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.base) + r * a.ld + c) = q;
  } else {
    float* p = reinterpret_cast<float*>(a.base) + r * a.ld + c;
    if constexpr (DT == DIPPM_DT_TF32X3) {
      float hi[8], lo[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        hi[i] = tf32_hi(v[i]);
        lo[i] = tf32_rn(v[i] - hi[i]);
      }
      reinterpret_cast<float4*>(p)[0] = make_float4(hi[0], hi[1], hi[2], hi[3]);
      reinterpret_cast<float4*>(p)[1] = make_float4(hi[4], hi[5], hi[6], hi[7]);
      reinterpret_cast<float4*>(p + a.plane_stride)[0] = make_float4(lo[0], lo[1], lo[2], lo[3]);
      reinterpret_cast<float4*>(p + a.plane_stride)[1] = make_float4(lo[4], lo[5], lo[6], lo[7]);
    } else {
      reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
      reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
    }
  }
}

// Sum of one double per thread over a 256-thread block in a fixed order (xor-shuffle tree in
// each warp, then the 8 warp sums in warp order by thread 0): deterministic, and ~10 dependent
// steps instead of a 256-long serial loop.  Result valid in thread 0.  s: >= 8 doubles of
// shared memory; every thread of the block must call it.
__device__ __forceinline__ double block_sum256(double v, double* s) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
#pragma unroll
    for (int w = 0; w < 8; ++w) t += s[w];
  __syncthreads();
  return t;
}

inline ActView make_view(const dippm_act_t& a) {
  ActView v;
  v.base = a.data;
  v.ld = a.ld;
  v.plane_stride = a.plane_stride;
  v.dtype = a.dtype;
  return v;
}

// mig.py:32-45 — one rule for host and device.  Ceilings 5/10/20/40 GiB in MB
// (1 GB = 1024 MB, mig.py:19-22), upper bounds inclusive, <=0 or >40960 -> None.
__host__ __device__ __forceinline__ int mig_rule(double a) {
  if (!(a > 0.0)) return -1;
  if (a <= 5120.0) return 0;
  if (a <= 10240.0) return 1;
  if (a <= 20480.0) return 2;
  if (a <= 40960.0) return 3;
  return -1;
}

// Counter-based dropout hash (train-mode throughput path; statistical parity
// with numerics.py:45-55, not bit parity — bit parity uses host-drawn masks).
__device__ __forceinline__ float uniform_hash(uint64_t seed, uint64_t counter) {
  uint64_t z = seed + 0x9E3779B97F4A7C15ull * (counter + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z = z ^ (z >> 31);
  return (float)(z >> 40) * (1.0f / 16777216.0f);
}

}  // namespace dippm
