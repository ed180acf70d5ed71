// K5/K6 fused — the whole FC head of a training step (fc1 -> fc2 -> fc3 -> Huber ->
// fc3/fc2/fc1 backward) in ONE persistent cooperative launch, for the small batches of
// training (G <= 576 graphs per rank, hidden <= 512, bf16 operands).
//
// At G = 256 the head is 0.3 % of a step's FLOPs but ran as 6 tensor-core GEMM launches
// and 5 small kernels (~115 us of an 800 us step): each of those GEMMs has 16-32 tiles
// and walks a serial chain of L2 round trips.  Here every phase is cut into 32 x 32
// output tiles spread over all SMs (warp-level mma.sync m16n8k16, bf16 in / fp32
// accumulate, whole-K operand tiles staged by cp.async), phases separated by grid
// barriers:
//
//   A  x2 = drop(relu(u @ W1 + b1))          (+ 1-bit x2 > 0 masks)      gnn.py:274-281
//   B  x3 = drop(relu(x2 @ W2 + b2))                                     gnn.py:274-281
//   C  per graph (warp per row): out = x3 @ W3 + b3, de-normalise + MIG  gnn.py:282-284, 93
//      (predict), Huber + dout (numerics.py:58-73), d2 = (dout W3^T) * (x3 > 0) * keep
//   D  d1 = (d2 @ W2^T) * [x2 > 0] * keep, dW2 = x2^T d2, dW3 = x3^T dout,  gnn.py:293-298
//      db2 = sum d2, db3 = sum dout, loss / APE sums
//   E  dW1 = u^T d1, db1 = sum d1, du = d1 @ W1^T (sage: the readout gradient)
// With gw1 / gw2 NULL the dW2 / dW1 units are left to the caller (the training step runs them
// as tcgen05 weight-gradient GEMMs beside the backward): D and E then hold one wave of units
// each, on the critical path only what the readout backward needs.
//
// Every reduction runs in a fixed order (no atomics on values): results are deterministic.
// Dropout in generated mode uses the same counter hash and index as the GEMM epilogue
// (tc_gemm.cu), so both paths draw identical masks.
#include "common.cuh"

namespace dippm {
namespace hf {

constexpr int kThreads = 256;   // 8 warps: 2 (m16) x 4 (n8) warp tiles of a 32 x 32 tile
constexpr int kT = 32;          // output tile edge
constexpr int kMaxK = 576;      // u_width (hidden + 64) or G
constexpr int kPad = 8;         // bf16 elements of padding per smem row (ldmatrix bank spread)

struct Args {
  int G, hp, uw;
  const __nv_bfloat16 *u, *w1, *w2;
  const float *b1, *b2, *w3, *b3;
  __nv_bfloat16 *x2, *x3;
  uint32_t* bits;
  int64_t bits_ld;
  int drop_mode;
  float drop_p, keep_scale;
  uint64_t seed1, seed2;
  const int64_t* seed_dev;
  const float *mask1, *mask2;
  float* out;
  const double* norm;
  double* y_pred;
  int8_t* mig;
  int* nonfinite;
  const double* y_raw;
  double delta, grad_den;
  double* loss_out;
  float* dout;
  __nv_bfloat16 *d2, *d1;
  float *d2f, *d1f;
  double* row_loss;
  float *gw1, *gb1, *gw2, *gb2, *gw3, *gb3, *du;
  int* sync;
  int train;
  int defer_reduce;  // the column-sum / loss units run in k_head_reduce (dippm_head_reduce) instead
  const float *pool_part, *pool_graph;
  const double* fs_raw;  // phase 0 (optional): u from the readout's block sums
  const int* graph_ptr;
  long long* step_counter;  // incremented in phase E (after every CTA's dropout draws)
};

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ int ld_acq(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// diagnostics: SM clock of CTA 0 at kernel start and, per phase, when its first unit's
// operands landed / that unit was done / its last unit was done / the grid barrier opened
constexpr int kTrace = 24;
__device__ long long g_trace[kTrace];
__device__ __forceinline__ void stamp(int i) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && i < kTrace) g_trace[i] = clock64();
}

// Grid barrier on {count, generation}.  Thread 0 of every CTA reads the generation once at
// kernel start (g0; the previous launch has completed, so all CTAs see the same value);
// barrier k of this launch opens when the generation reaches g0 + k + 1, which the last
// arriver publishes (after returning count to 0, so the pair is ready for the next barrier
// and the next launch: graph replays need no reset).  One atomic round trip per CTA, then
// acquire polls; the release/acquire pair orders each phase's writes before the next phase.
struct GridBar {
  int* count;
  int* gen;
  int g0, k;
  __device__ void init(int* sync) {
    count = sync;
    gen = sync + 1;
    k = 0;
    if (threadIdx.x == 0) g0 = ld_acq(gen);
  }
  __device__ void sync() {
    __syncthreads();
    ++k;
    if (threadIdx.x == 0) {
      const int target = g0 + k;
      __threadfence();  // this CTA's phase writes (ordered by the bar.sync) before the arrival
      if (atomicAdd(count, 1) == (int)gridDim.x - 1) {
        asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(count), "r"(0) : "memory");
        st_rel(gen, target);
      } else {
        uint32_t spins = 0;
        uint64_t t0 = 0;
        while (ld_acq(gen) - target < 0) {
          if (++spins == 64) t0 = gtimer();
          if (spins > 64 && (spins & 255) == 0 && gtimer() - t0 > 2000000000ull) __trap();  // co-residency bug
        }
      }
    }
    __syncthreads();
  }
};

// 16-byte async copy; src_bytes = 0 zero-fills (rows past the end of a matrix).
__device__ __forceinline__ void cp16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(su32(dst)), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// rows [r0, r0 + nr) x cols [c0, c0 + nc) of a row-major bf16 matrix (ld elements) into
// smem rows of sld elements; rows >= rmax read as zero.  nc % 8 == 0.
__device__ __forceinline__ void load_tile(__nv_bfloat16* s, int sld, const __nv_bfloat16* g, int64_t ld, int r0,
                                          int nr, int rmax, int c0, int nc) {
  const int cpr = nc >> 3;
  for (int i = threadIdx.x; i < nr * cpr; i += kThreads) {
    const int r = i / cpr, c = (i - r * cpr) << 3;
    const bool ok = r0 + r < rmax;
    cp16(s + r * sld + c, g + (int64_t)(ok ? r0 + r : 0) * ld + c0 + c, ok ? 16 : 0);
  }
}

__device__ __forceinline__ void ldm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(su32(p)));
}
__device__ __forceinline__ void ldm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(su32(p)));
}
__device__ __forceinline__ void ldm_x2(uint32_t& r0, uint32_t& r1, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(su32(p)));
}
__device__ __forceinline__ void ldm_x2_t(uint32_t& r0, uint32_t& r1, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(su32(p)));
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// One 32 x 32 tile C = sum_k A(m, k) B(k, n), K (a multiple of 32) split over the 8 warps:
// warp w takes the k16 steps s = w, w + 8, ... and accumulates the whole tile (2 m16 x 4 n8
// fragments, 8 independent mma chains); the partials meet in shared memory and every
// thread sums its 4 outputs over the warps in warp order (fixed order: deterministic).
// kAkm: A staged as [k][m] (else [m][k]); kBkn: B staged as [k][n] (else [n][k]).
// On return thread t holds row t / 8, columns 4 (t % 8) .. + 3 in out[4].
constexpr int kRedLd = kT + 4;  // fp32 row stride of the reduction scratch (16 B aligned rows)
template <bool kAkm, bool kBkn>
__device__ __forceinline__ void cta_tile(const __nv_bfloat16* sA, int lda, const __nv_bfloat16* sB, int ldb, int K,
                                         float* red, float (&out)[4]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float acc[2][4][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.f;
  // per-lane ldmatrix row addresses at k = 0 for the two m16 blocks / two n16 pairs
  const __nv_bfloat16 *pa0, *pa1, *pb0, *pb1;
  int sa, sb;  // element step per k16
  if constexpr (kAkm) {
    const int r = (lane & 7) + ((lane >> 4) << 3), c = ((lane >> 3) & 1) << 3;
    pa0 = sA + r * lda + c;
    pa1 = pa0 + 16;
    sa = 16 * lda;
  } else {
    const int r = lane & 15, c = (lane >> 4) << 3;
    pa0 = sA + r * lda + c;
    pa1 = pa0 + 16 * lda;
    sa = 16;
  }
  if constexpr (kBkn) {
    const int r = (lane & 7) + (((lane >> 3) & 1) << 3), c = (lane >> 4) << 3;
    pb0 = sB + r * ldb + c;
    pb1 = pb0 + 16;
    sb = 16 * ldb;
  } else {
    const int r = (lane & 7) + ((lane >> 4) << 3), c = ((lane >> 3) & 1) << 3;
    pb0 = sB + r * ldb + c;
    pb1 = pb0 + 16 * ldb;
    sb = 16;
  }
  for (int s = w; s < (K >> 4); s += 8) {
    uint32_t a[2][4], b[2][4];
    if constexpr (kAkm) {
      ldm_x4_t(a[0], pa0 + s * sa);
      ldm_x4_t(a[1], pa1 + s * sa);
    } else {
      ldm_x4(a[0], pa0 + s * sa);
      ldm_x4(a[1], pa1 + s * sa);
    }
    if constexpr (kBkn) {
      ldm_x4_t(b[0], pb0 + s * sb);
      ldm_x4_t(b[1], pb1 + s * sb);
    } else {
      ldm_x4(b[0], pb0 + s * sb);
      ldm_x4(b[1], pb1 + s * sb);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) mma_bf16(acc[i][j], a[i], b[j >> 1][(j & 1) * 2], b[j >> 1][(j & 1) * 2 + 1]);
  }
  float* my = red + w * kT * kRedLd;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = i * 16 + (lane >> 2) + h * 8, col = j * 8 + ((lane & 3) << 1);
        *reinterpret_cast<float2*>(my + row * kRedLd + col) = make_float2(acc[i][j][2 * h], acc[i][j][2 * h + 1]);
      }
  __syncthreads();
  const int row = threadIdx.x >> 3, col = (threadIdx.x & 7) << 2;
  float4 t = *reinterpret_cast<const float4*>(red + row * kRedLd + col);
#pragma unroll
  for (int q = 1; q < 8; ++q) {
    const float4 v = *reinterpret_cast<const float4*>(red + q * kT * kRedLd + row * kRedLd + col);
    t.x += v.x;
    t.y += v.y;
    t.z += v.z;
    t.w += v.w;
  }
  out[0] = t.x;
  out[1] = t.y;
  out[2] = t.z;
  out[3] = t.w;
}

__device__ __forceinline__ int round32(int x) { return (x + 31) & ~31; }

// ---- the unit pipeline -------------------------------------------------------
// A phase is a list of independent units (a 32 x 32 output tile, or a 32-column
// reduction).  Each CTA walks its units with a two-buffer cp.async pipeline: the operands
// of its next unit stream in while the current one computes.
enum UnitType { U_FWD1, U_FWD2, U_WG2, U_GATE, U_CS2, U_LOSS, U_WG1, U_STORE, U_CS1 };
struct Unit {
  int type, m0, n0;
};
constexpr int kBuf = 2 * kMaxK * (kT + kPad) * 2;  // bytes per operand buffer (A + B)
constexpr int kScratch = 8 * kT * kRedLd * 4;      // K-split partials (also the reduction units' scratch)
constexpr int kSmemTotal = 2 * kBuf + kScratch;

__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ __nv_bfloat16* buf_a(uint8_t* b) { return reinterpret_cast<__nv_bfloat16*>(b); }
__device__ __forceinline__ __nv_bfloat16* buf_b(uint8_t* b) { return buf_a(b) + kMaxK * (kT + kPad); }

// stage the operands of unit u into buffer b (asynchronous)
__device__ void issue(const Args& a, const Unit& u, uint8_t* b) {
  const int G32 = round32(a.G);
  switch (u.type) {
    case U_FWD1:
    case U_FWD2: {  // A = X [32 x K] (K-major), B = W [K x 32] (N contiguous)
      const int K = u.type == U_FWD1 ? a.uw : a.hp;
      load_tile(buf_a(b), K + kPad, u.type == U_FWD1 ? a.u : a.x2, K, u.m0, kT, a.G, 0, K);
      load_tile(buf_b(b), kT + kPad, u.type == U_FWD1 ? a.w1 : a.w2, a.hp, 0, K, K, u.n0, kT);
      break;
    }
    case U_WG2:
    case U_WG1: {  // A = X [G x 32] staged [k][m], B = D [G x 32] staged [k][n]
      const bool l2 = u.type == U_WG2;
      load_tile(buf_a(b), kT + kPad, l2 ? a.x2 : a.u, l2 ? a.hp : a.uw, 0, G32, a.G, u.m0, kT);
      load_tile(buf_b(b), kT + kPad, l2 ? a.d2 : a.d1, a.hp, 0, G32, a.G, u.n0, kT);
      break;
    }
    case U_GATE:
    case U_STORE: {  // A = D [32 x hp], B = W rows [n0, n0 + 32) x hp (= W^T staged [n][k])
      const bool g = u.type == U_GATE;
      load_tile(buf_a(b), a.hp + kPad, g ? a.d2 : a.d1, a.hp, u.m0, kT, a.G, 0, a.hp);
      load_tile(buf_b(b), a.hp + kPad, g ? a.w2 : a.w1, a.hp, u.n0, kT, 1 << 30, 0, a.hp);
      break;
    }
    default:
      break;  // reductions read global memory directly
  }
}

// x_out = drop(relu(acc + b)) for FWD1 (x2, + bit masks) / FWD2 (x3); this thread's
// row t / 8, columns 4 (t % 8) .. + 3 of the tile
__device__ void fwd_epilogue(const Args& a, const Unit& u, const float (&acc)[4]) {
  const bool l1 = u.type == U_FWD1;
  const float* bias = l1 ? a.b1 : a.b2;
  const float* mask = l1 ? a.mask1 : a.mask2;
  __nv_bfloat16* xout = l1 ? a.x2 : a.x3;
  uint64_t seed = l1 ? a.seed1 : a.seed2;
  if (a.drop_mode == 2 && a.seed_dev) seed ^= (uint64_t)a.seed_dev[0] * 0x9E3779B97F4A7C15ull;
  const float keep = 1.0f / (1.0f - a.drop_p);
  const int lc = (threadIdx.x & 7) << 2;
  const int row = u.m0 + (threadIdx.x >> 3), col = u.n0 + lc;
  const float4 b4 = *reinterpret_cast<const float4*>(bias + col);
  float v[4] = {fmaxf(acc[0] + b4.x, 0.f), fmaxf(acc[1] + b4.y, 0.f), fmaxf(acc[2] + b4.z, 0.f),
                fmaxf(acc[3] + b4.w, 0.f)};
  if (row < a.G) {
    const int64_t idx = (int64_t)row * a.hp + col;
    if (a.drop_mode == 1) {
      const float4 m4 = *reinterpret_cast<const float4*>(mask + idx);
      v[0] *= m4.x;
      v[1] *= m4.y;
      v[2] *= m4.z;
      v[3] *= m4.w;
    } else if (a.drop_mode == 2) {  // tc_gemm.cu's counter hash and index
#pragma unroll
      for (int i = 0; i < 4; ++i) v[i] *= uniform_hash(seed, (uint64_t)(idx + i)) >= a.drop_p ? keep : 0.f;
    }
    __nv_bfloat162 h[2] = {__floats2bfloat162_rn(v[0], v[1]), __floats2bfloat162_rn(v[2], v[3])};
    *reinterpret_cast<uint2*>(xout + idx) = *reinterpret_cast<uint2*>(h);
  }
  if (l1 && a.bits) {  // the 8 lanes of a row OR their nibbles into the row's 32-bit word
    uint32_t word = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) word |= (uint32_t)(v[i] > 0.f) << (lc + i);
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) word |= __shfl_xor_sync(0xffffffffu, word, o);
    if ((threadIdx.x & 7) == 0 && row < a.G) a.bits[(int64_t)(u.n0 >> 5) * a.bits_ld + row] = word;
  }
}

// ---- column sums of kCsCols columns over the G rows (32 row groups, fixed order) ----
// what: 0 = db2 (d2f) + dW3 (x3^T dout), 1 = db1 (d1f).  Narrow units, many row groups: each
// thread's rows (G / 32 of them, written this launch by other CTAs) load in one batch of L2
// reads for G <= 256; 32 columns x 8 row groups was a chain of G / 64 dependent round trips
// and the longest unit of phases D / E.
constexpr int kCsCols = 8;
__device__ void colsum_unit(const Args& a, uint8_t* smem, int what, int c0) {  // smem: scratch
  float(*s)[kCsCols][4] = reinterpret_cast<float(*)[kCsCols][4]>(smem);  // [32][kCsCols][4]
  const int tx = threadIdx.x % kCsCols, ty = threadIdx.x / kCsCols, j = c0 + tx;
  const float* src = what == 0 ? a.d2f : a.d1f;
  float cb = 0.f, w0 = 0.f, w1 = 0.f, w2 = 0.f;
  for (int g0 = ty; g0 < a.G; g0 += 32 * 8) {  // rows g0, g0 + 32, ... (8 per batch)
    float sv[8], xv[8], dv[8][3];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int g = g0 + 32 * i;
      const bool ok = g < a.G;
      sv[i] = ok ? __ldcg(src + (int64_t)g * a.hp + j) : 0.f;
      if (what == 0) {
        xv[i] = ok ? __bfloat162float(__ldcg(a.x3 + (int64_t)g * a.hp + j)) : 0.f;
#pragma unroll
        for (int k = 0; k < 3; ++k) dv[i][k] = ok ? __ldcg(a.dout + g * 3 + k) : 0.f;
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (g0 + 32 * i >= a.G) break;
      cb += sv[i];
      if (what == 0) {
        w0 = fmaf(xv[i], dv[i][0], w0);
        w1 = fmaf(xv[i], dv[i][1], w1);
        w2 = fmaf(xv[i], dv[i][2], w2);
      }
    }
  }
  s[ty][tx][0] = cb;
  s[ty][tx][1] = w0;
  s[ty][tx][2] = w1;
  s[ty][tx][3] = w2;
  __syncthreads();
  if (threadIdx.x < kCsCols) {
    float r[4] = {0.f, 0.f, 0.f, 0.f};
    for (int q = 0; q < 32; ++q)
      for (int k = 0; k < 4; ++k) r[k] += s[q][tx][k];
    if (what == 0) {
      a.gb2[j] = r[0];
      a.gw3[j * 3 + 0] = r[1];
      a.gw3[j * 3 + 1] = r[2];
      a.gw3[j * 3 + 2] = r[3];
    } else {
      a.gb1[j] = r[0];
    }
  }
  __syncthreads();
}

// ---- batch loss (k_huber's reduction order: per-thread strided sums, then block_sum256) and db3 ----
__device__ void loss_unit(const Args& a, uint8_t* smem) {
  double* sw = reinterpret_cast<double*>(smem);  // [8]
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  float b[3] = {0.f, 0.f, 0.f};
  for (int g = threadIdx.x; g < a.G; g += kThreads) {
    for (int k = 0; k < 4; ++k) acc[k] += __ldcg(a.row_loss + (int64_t)g * 4 + k);
    if (a.train)
      for (int k = 0; k < 3; ++k) b[k] += __ldcg(a.dout + g * 3 + k);
  }
  double t[4];
  for (int k = 0; k < 4; ++k) t[k] = block_sum256(acc[k], sw);
  float tb[3] = {0.f, 0.f, 0.f};
  if (a.train) {
    // db3 in fp32, fixed order: xor tree per warp, warps in order
    float* sf = reinterpret_cast<float*>(sw + 8);  // [8][3]
    for (int k = 0; k < 3; ++k) {
      float v = b[k];
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if ((threadIdx.x & 31) == 0) sf[(threadIdx.x >> 5) * 3 + k] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int w = 0; w < 8; ++w)
        for (int k = 0; k < 3; ++k) tb[k] += sf[w * 3 + k];
  }
  if (threadIdx.x == 0) {
    a.loss_out[0] = t[0] / (double)a.G;
    for (int k = 0; k < 3; ++k) a.loss_out[1 + k] = t[1 + k];
    if (a.train)
      for (int k = 0; k < 3; ++k) a.gb3[k] = tb[k];
  }
  __syncthreads();
}

// compute unit u from buffer b (its operands have landed)
__device__ void run(const Args& a, const Unit& u, uint8_t* b, uint8_t* scratch) {
  float* red = reinterpret_cast<float*>(scratch);
  float acc[4];
  const int row = u.m0 + (threadIdx.x >> 3), col = u.n0 + ((threadIdx.x & 7) << 2);
  switch (u.type) {
    case U_FWD1:
    case U_FWD2: {
      const int K = u.type == U_FWD1 ? a.uw : a.hp;
      cta_tile<false, true>(buf_a(b), K + kPad, buf_b(b), kT + kPad, K, red, acc);
      fwd_epilogue(a, u, acc);
      break;
    }
    case U_WG2:
    case U_WG1: {  // dW = X^T D (fixed K order), straight to the fp32 gradient
      cta_tile<true, true>(buf_a(b), kT + kPad, buf_b(b), kT + kPad, round32(a.G), red, acc);
      float* gw = u.type == U_WG2 ? a.gw2 : a.gw1;
      *reinterpret_cast<float4*>(gw + (int64_t)row * a.hp + col) = make_float4(acc[0], acc[1], acc[2], acc[3]);
      break;
    }
    case U_GATE:
    case U_STORE: {
      cta_tile<false, false>(buf_a(b), a.hp + kPad, buf_b(b), a.hp + kPad, a.hp, red, acc);
      if (row >= a.G) break;
      const int64_t idx = (int64_t)row * a.hp + col;
      if (u.type == U_GATE) {  // d1 = (d2 W2^T) * [x2 > 0] * keep, on the forward's bits
        const uint32_t word = a.bits[(int64_t)(col >> 5) * a.bits_ld + row] >> (col & 31);
        float v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = (word >> i) & 1u ? acc[i] * a.keep_scale : 0.f;
        __nv_bfloat162 h[2] = {__floats2bfloat162_rn(v[0], v[1]), __floats2bfloat162_rn(v[2], v[3])};
        *reinterpret_cast<uint2*>(a.d1 + idx) = *reinterpret_cast<uint2*>(h);
        *reinterpret_cast<float4*>(a.d1f + idx) = make_float4(v[0], v[1], v[2], v[3]);
      } else {  // du = d1 W1^T (readout columns)
        *reinterpret_cast<float4*>(a.du + idx) = make_float4(acc[0], acc[1], acc[2], acc[3]);
      }
      break;
    }
    case U_CS2:
      colsum_unit(a, scratch, 0, u.n0);
      break;
    case U_CS1:
      colsum_unit(a, scratch, 1, u.n0);
      break;
    case U_LOSS:
      loss_unit(a, scratch);
      break;
  }
}

template <class UnitOf>
__device__ void run_phase(const Args& a, uint8_t* smem, int n, UnitOf unit_of, int tr) {
  int t = blockIdx.x, buf = 0;
  if (t < n) issue(a, unit_of(t), smem);
  cp_commit();
  for (; t < n; t += gridDim.x) {
    const int tn = t + gridDim.x;
    if (tn < n) issue(a, unit_of(tn), smem + (buf ^ 1) * kBuf);
    cp_commit();
    cp_wait<1>();  // this unit's group has landed (the next one may still be in flight)
    __syncthreads();
    if (t == 0) stamp(tr);
    run(a, unit_of(t), smem + buf * kBuf, smem + 2 * kBuf);
    __syncthreads();  // buffer `buf` is free for the unit after next
    if (t == 0) stamp(tr + 1);
    buf ^= 1;
  }
  cp_wait<0>();
  stamp(tr + 2);
}

// ---- phase C: one warp per graph row ----
__device__ void head_rows(const Args& a) {
  // each lane owns 8-column chunks lane and lane + 32 of the row (hp <= 512): all of its x3
  // and W3 operands are loaded in one go (one latency), d2 is stored 8 columns at a time
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (kThreads / 32);
  const int nch = a.hp >> 3;
  for (int g = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); g < a.G; g += warps) {
    const __nv_bfloat16* xr = a.x3 + (int64_t)g * a.hp;
    float x[2][8], w[2][24];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int c = lane + 32 * q;
      if (c < nch) {
        const uint4 xv = __ldcg(reinterpret_cast<const uint4*>(xr + c * 8));  // written this launch
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&xv);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = __bfloat1622float2(h[i]);
          x[q][2 * i] = f.x;
          x[q][2 * i + 1] = f.y;
        }
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(a.w3 + c * 24) + i);
          w[q][4 * i] = v.x;
          w[q][4 * i + 1] = v.y;
          w[q][4 * i + 2] = v.z;
          w[q][4 * i + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[q][i] = 0.f;
#pragma unroll
        for (int i = 0; i < 24; ++i) w[q][i] = 0.f;
      }
    }
    float s0 = 0.f, s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        s0 = fmaf(x[q][i], w[q][3 * i + 0], s0);
        s1 = fmaf(x[q][i], w[q][3 * i + 1], s1);
        s2 = fmaf(x[q][i], w[q][3 * i + 2], s2);
      }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    const float o3[3] = {s0 + a.b3[0], s1 + a.b3[1], s2 + a.b3[2]};
    float e[3] = {0.f, 0.f, 0.f};
    // lanes 0..2 each take one output column (the fp64 divisions of the three run in parallel)
    const float ok = lane == 0 ? o3[0] : (lane == 1 ? o3[1] : o3[2]);
    double le_k = 0.0;
    if (lane < 3) {
      const int k = lane;
      a.out[g * 3 + k] = ok;
      if (a.y_pred) a.y_pred[g * 3 + k] = (double)ok * a.norm[3 + k] + a.norm[k];
      if (a.y_raw) {  // k_huber's per-graph terms (head.cu)
        const double pred = (double)ok, y = a.y_raw[g * 3 + k];
        const double t = (y - a.norm[k]) / a.norm[3 + k];
        const double r = pred - t, ab = fabs(r);
        const bool quad = ab <= a.delta;
        le_k = quad ? 0.5 * r * r : a.delta * (ab - 0.5 * a.delta);
        const double gr = quad ? r : a.delta * (r > 0 ? 1.0 : (r < 0 ? -1.0 : 0.0));
        e[k] = (float)(gr / 3.0 / a.grad_den);
        if (a.dout) a.dout[g * 3 + k] = e[k];
        const double den = pred * a.norm[3 + k] + a.norm[k];
        a.row_loss[(int64_t)g * 4 + 1 + k] = fabs(den - y) / fabs(y);
      }
    }
    if (a.y_pred && lane == 1) {  // the memory column picks the MIG profile
      const double mem = (double)ok * a.norm[4] + a.norm[1];
      if (!isfinite(mem)) {
        atomicExch(a.nonfinite, 1);
        a.mig[g] = -1;
      } else {
        a.mig[g] = (int8_t)mig_rule(mem);
      }
    }
    if (a.y_raw) {  // le = ((l0 + l1) + l2) / 3, k_huber's order
      const double l1 = __shfl_sync(0xffffffffu, le_k, 1), l2 = __shfl_sync(0xffffffffu, le_k, 2);
      if (lane == 0) a.row_loss[(int64_t)g * 4] = ((0.0 + le_k) + l1 + l2) / 3.0;
    }
    if (!a.train) continue;
#pragma unroll
    for (int k = 0; k < 3; ++k) e[k] = __shfl_sync(0xffffffffu, e[k], k);
#pragma unroll
    for (int q = 0; q < 2; ++q) {  // d2 = (dout W3^T) * [x3 > 0] * keep (k_fc3_backward, head.cu)
      const int c = lane + 32 * q;
      if (c >= nch) continue;
      float dv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float dx = e[0] * w[q][3 * i] + e[1] * w[q][3 * i + 1] + e[2] * w[q][3 * i + 2];
        dv[i] = x[q][i] > 0.f ? dx * a.keep_scale : 0.f;
      }
      const int64_t o = (int64_t)g * a.hp + c * 8;
      __nv_bfloat162 h[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(dv[2 * i], dv[2 * i + 1]);
      *reinterpret_cast<uint4*>(a.d2 + o) = *reinterpret_cast<uint4*>(h);
      *reinterpret_cast<float4*>(a.d2f + o) = make_float4(dv[0], dv[1], dv[2], dv[3]);
      *reinterpret_cast<float4*>(a.d2f + o + 4) = make_float4(dv[4], dv[5], dv[6], dv[7]);
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1) k_head_fused(Args a) {
  extern __shared__ __align__(16) uint8_t smem[];
  stamp(0);
  GridBar bar;
  bar.init(a.sync);
  const int mt = (a.G + kT - 1) / kT, nh = a.hp / kT, nu = a.uw / kT;
  if (a.pool_part) {
    // 0: u = [mean of the layer-3 rows | (fs - mu) / sigma | 0], dippm_pool_combine's
    // arithmetic (fp64 block sums in block order, bf16), one graph per CTA at a time
    __nv_bfloat16* u = const_cast<__nv_bfloat16*>(a.u);
    for (int g = blockIdx.x; g < a.G; g += gridDim.x) {
      const int gs = a.graph_ptr[g], ge = a.graph_ptr[g + 1];
      const int bf = gs >> 5, bl = (ge - 1) >> 5;
      const double inv_n = 1.0 / (double)(ge - gs);
      for (int c = threadIdx.x; c < a.hp; c += kThreads) {
        double t;
        if (bf == bl) {
          t = a.pool_graph[(int64_t)g * a.hp + c];
        } else {
          t = a.pool_part[((int64_t)bf * 2 + ((gs & 31) == 0 ? 0 : 1)) * a.hp + c];
          int b = bf + 1;
          for (; b + 4 <= bl; b += 4) {
            const float v0 = a.pool_part[(int64_t)b * 2 * a.hp + c], v1 = a.pool_part[(int64_t)(b + 1) * 2 * a.hp + c];
            const float v2 = a.pool_part[(int64_t)(b + 2) * 2 * a.hp + c];
            const float v3 = a.pool_part[(int64_t)(b + 3) * 2 * a.hp + c];
            t += v0;
            t += v1;
            t += v2;
            t += v3;
          }
          for (; b < bl; ++b) t += a.pool_part[(int64_t)b * 2 * a.hp + c];
          t += a.pool_part[(int64_t)bl * 2 * a.hp + c];
        }
        u[(int64_t)g * a.uw + c] = __float2bfloat16_rn((float)(t * inv_n));
      }
      for (int k = threadIdx.x; k < a.uw - a.hp; k += kThreads) {
        float v = 0.f;
        if (k < kStaticWidth) v = (float)((a.fs_raw[g * kStaticWidth + k] - a.norm[6 + k]) / a.norm[11 + k]);
        u[(int64_t)g * a.uw + a.hp + k] = __float2bfloat16_rn(v);
      }
    }
    bar.sync();
  }
  // A, B: the two hidden layers
  run_phase(a, smem, mt * nh, [&](int t) { return Unit{U_FWD1, (t / nh) * kT, (t % nh) * kT}; }, 1);
  bar.sync();
  stamp(4);
  run_phase(a, smem, mt * nh, [&](int t) { return Unit{U_FWD2, (t / nh) * kT, (t % nh) * kT}; }, 5);
  bar.sync();
  stamp(8);
  // C: fc3, output stage, per-graph loss terms, d2
  head_rows(a);
  stamp(9);
  if (!a.y_raw) return;
  bar.sync();
  stamp(10);
  // D: dW2, GATE d1, db2 + dW3, loss + db3 (longest units first)
  {
    const int n_w = a.train && a.gw2 ? nh * nh : 0, n_g = a.train ? mt * nh : 0;
    const int n_c = a.train && !a.defer_reduce ? a.hp / kCsCols : 0, n_l = a.defer_reduce ? 0 : 1;
    run_phase(a, smem, n_w + n_g + n_c + n_l, [&](int t) {
      if (t < n_w) return Unit{U_WG2, (t / nh) * kT, (t % nh) * kT};
      t -= n_w;
      if (t < n_g) return Unit{U_GATE, (t / nh) * kT, (t % nh) * kT};
      t -= n_g;
      if (t < n_c) return Unit{U_CS2, 0, t * kCsCols};
      return Unit{U_LOSS, 0, 0};
    }, 11);
  }
  if (!a.train) return;
  bar.sync();
  stamp(14);
  if (a.step_counter && blockIdx.x == 0 && threadIdx.x == 0) a.step_counter[0] += 1;  // phases A/B are done
  // E: dW1, du, db1
  {
    const int n_w = a.gw1 ? nu * nh : 0, n_s = a.du ? mt * nh : 0;  // (gw1 NULL: dW1 by the caller)
    const int n_c = a.defer_reduce ? 0 : a.hp / kCsCols;
    run_phase(a, smem, n_w + n_s + n_c, [&](int t) {
      if (t < n_w) return Unit{U_WG1, (t / nh) * kT, (t % nh) * kT};
      t -= n_w;
      if (t < n_s) return Unit{U_STORE, (t / nh) * kT, (t % nh) * kT};
      t -= n_s;
      return Unit{U_CS1, 0, t * kCsCols};
    }, 15);
  }
  // no closing grid barrier: the kernel's completion orders phase E's writes for the next
  // launch, and the barrier pair is already reset (the last arriver of D returned count to 0)
  stamp(18);
}

// The head's reductions as their own launch (training step, side stream): db2 + dW3 and db1
// column sums (colsum_unit) and the batch loss + db3 (loss_unit) -- the same units, so the
// same results as inside k_head_fused; one unit per CTA.
__global__ void __launch_bounds__(kThreads) k_head_reduce(const Args a) {
  __shared__ __align__(16) uint8_t scratch[32 * kCsCols * 4 * 4];
  const int nc = a.hp / kCsCols;
  const int t = blockIdx.x;
  if (t < nc) colsum_unit(a, scratch, 0, t * kCsCols);
  else if (t < 2 * nc) colsum_unit(a, scratch, 1, (t - nc) * kCsCols);
  else loss_unit(a, scratch);
}

}  // namespace hf
}  // namespace dippm

using namespace dippm;

namespace dippm {
bool head_tc_launch(const dippm_head_args_t* h, cudaStream_t s, int32_t* status);  // head_tc.cu
int head_tc_trace(unsigned long long* out16);
// the tensor-core head (head_tc.cu) for the shapes it covers: opt-in, DIPPM_HEAD_TC=1 or
// dippm_head_tc_enable(1) -- it measured ~4x slower than this kernel at configs[1]
static int g_head_tc = -1;
static bool head_tc_enabled() {
  if (g_head_tc < 0) g_head_tc = getenv("DIPPM_HEAD_TC") && getenv("DIPPM_HEAD_TC")[0] == '1';
  return g_head_tc != 0;
}
}

namespace dippm {
static hf::Args head_args(const dippm_head_args_t* h) {
  hf::Args a{};
  a.G = (int)h->G;
  a.hp = h->hp;
  a.uw = h->u_width;
  a.u = reinterpret_cast<const __nv_bfloat16*>(h->u);
  a.w1 = reinterpret_cast<const __nv_bfloat16*>(h->w1);
  a.w2 = reinterpret_cast<const __nv_bfloat16*>(h->w2);
  a.b1 = h->b1;
  a.b2 = h->b2;
  a.w3 = h->w3;
  a.b3 = h->b3;
  a.x2 = reinterpret_cast<__nv_bfloat16*>(h->x2);
  a.x3 = reinterpret_cast<__nv_bfloat16*>(h->x3);
  a.bits = h->bits;
  a.bits_ld = h->bits_ld;
  a.drop_mode = h->drop_mode;
  a.drop_p = (float)h->drop_p;
  a.keep_scale = h->keep_scale;
  a.seed1 = h->seed1;
  a.seed2 = h->seed2;
  a.seed_dev = h->seed_dev;
  a.mask1 = h->mask1;
  a.mask2 = h->mask2;
  a.out = h->out;
  a.norm = h->norm;
  a.y_pred = h->y_pred;
  a.mig = h->mig;
  a.nonfinite = h->nonfinite;
  a.y_raw = h->y_raw;
  a.delta = h->delta;
  a.grad_den = h->grad_den > 0 ? h->grad_den : (double)h->G;
  a.loss_out = h->loss_out;
  a.dout = h->dout;
  a.d2 = reinterpret_cast<__nv_bfloat16*>(h->d2);
  a.d1 = reinterpret_cast<__nv_bfloat16*>(h->d1);
  a.d2f = h->d2f;
  a.d1f = h->d1f;
  a.row_loss = h->row_loss;
  a.gw1 = h->gw1;
  a.gb1 = h->gb1;
  a.gw2 = h->gw2;
  a.gb2 = h->gb2;
  a.gw3 = h->gw3;
  a.gb3 = h->gb3;
  a.du = h->du;
  a.sync = h->sync;
  a.train = h->train ? 1 : 0;
  a.pool_part = h->pool_partial;
  a.pool_graph = h->pool_graph;
  a.graph_ptr = h->graph_ptr;
  a.fs_raw = h->fs_raw;
  a.step_counter = reinterpret_cast<long long*>(h->step_counter);
  a.defer_reduce = h->defer_reduce ? 1 : 0;
  return a;
}

}  // namespace dippm

extern "C" {

int32_t dippm_head_fused_max_graphs(void) { return hf::kMaxK; }
int32_t dippm_head_fused_sync_ints(void) { return 2; }  // the grid barrier's {count, generation}
int32_t dippm_head_tc_trace(uint64_t* out16) { return head_tc_trace(reinterpret_cast<unsigned long long*>(out16)); }
int32_t dippm_head_tc_enable(int32_t on) {
  const int32_t was = head_tc_enabled() ? 1 : 0;
  if (on >= 0) g_head_tc = on ? 1 : 0;
  return was;
}

int32_t dippm_head_fused_trace(int64_t* out24) {
  long long t[hf::kTrace];
  DIPPM_CUDA_CHECK(cudaMemcpyFromSymbol(t, hf::g_trace, sizeof(t)));
  for (int i = 0; i < hf::kTrace; ++i) out24[i] = (int64_t)(t[i] - t[0]);
  return DIPPM_OK;
}

int32_t dippm_head_fused(const dippm_head_args_t* h, void* stream) {
  DIPPM_ARG_CHECK(h && h->G >= 1 && h->G <= hf::kMaxK, "head_fused: G must be in [1, %d]", hf::kMaxK);
  DIPPM_ARG_CHECK(h->hp >= 32 && h->hp % 64 == 0 && h->hp <= 512, "head_fused: hidden width must be a multiple of 64 <= 512");
  DIPPM_ARG_CHECK(h->u_width % 64 == 0 && h->u_width >= 64 && h->u_width <= hf::kMaxK, "head_fused: bad u_width");
  DIPPM_ARG_CHECK(h->u && h->w1 && h->w2 && h->b1 && h->b2 && h->w3 && h->b3 && h->x2 && h->x3 && h->out && h->sync,
                  "head_fused: missing operand");
  DIPPM_ARG_CHECK(!h->bits || h->bits_ld >= h->G, "head_fused: bits_ld < G");
  DIPPM_ARG_CHECK(!h->pool_partial || (h->pool_graph && h->graph_ptr && h->fs_raw && h->norm &&
                                       h->u_width >= h->hp + kStaticWidth),
                  "head_fused: in-kernel readout needs pool_graph, graph_ptr, fs_raw, norm, u_width >= hp + 5");
  DIPPM_ARG_CHECK(h->drop_mode >= 0 && h->drop_mode <= 2 && h->drop_p >= 0 && h->drop_p < 1,
                  "head_fused: bad dropout arguments");
  DIPPM_ARG_CHECK(h->drop_mode != 1 || (h->mask1 && h->mask2), "head_fused: dropout mode 1 needs both masks");
  DIPPM_ARG_CHECK(!h->y_pred || (h->norm && h->mig && h->nonfinite), "head_fused: y_pred needs norm, mig, nonfinite");
  DIPPM_ARG_CHECK(!h->y_raw || (h->norm && h->loss_out && h->row_loss && h->delta > 0),
                  "head_fused: loss needs norm, loss_out, row_loss, delta > 0");
  DIPPM_ARG_CHECK(!h->train || (h->y_raw && h->bits && h->dout && h->d1 && h->d2 && h->d1f && h->d2f &&
                                h->gb1 && h->gb2 && h->gw3 && h->gb3 && (h->gw1 != nullptr) == (h->gw2 != nullptr)),
                  "head_fused: training needs targets, bit masks, gradient buffers");
  // opt-in: the configs[1] head (G <= 256, hidden 512, training step) on the tensor cores (head_tc.cu)
  int32_t st = DIPPM_OK;
  if (head_tc_enabled() && head_tc_launch(h, (cudaStream_t)stream, &st)) return st;
  const hf::Args a = head_args(h);
  static bool attr = false;
  if (!attr) {
    DIPPM_CUDA_CHECK(cudaFuncSetAttribute(hf::k_head_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          hf::kSmemTotal));
    attr = true;
  }
  // one CTA per SM, all co-resident (cooperative launch: the grid barriers need it)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)num_sms());
  cfg.blockDim = dim3(hf::kThreads);
  cfg.dynamicSmemBytes = hf::kSmemTotal;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  DIPPM_CUDA_CHECK(cudaLaunchKernelEx(&cfg, hf::k_head_fused, a));
  DIPPM_LAUNCH_CHECK("k_head_fused");
  return DIPPM_OK;
}

int32_t dippm_head_reduce(const dippm_head_args_t* h, void* stream) {
  DIPPM_ARG_CHECK(h && h->train && h->defer_reduce && h->G >= 1 && h->hp % hf::kCsCols == 0 && h->d1f &&
                      h->d2f && h->x3 && h->dout && h->row_loss && h->loss_out && h->gb1 && h->gb2 && h->gw3 &&
                      h->gb3,
                  "head_reduce: needs the training head's arguments with defer_reduce set");
  const hf::Args a = head_args(h);
  hf::k_head_reduce<<<2 * (h->hp / hf::kCsCols) + 1, hf::kThreads, 0, (cudaStream_t)stream>>>(a);
  DIPPM_LAUNCH_CHECK("k_head_reduce");
  return DIPPM_OK;
}

}  // extern "C"
