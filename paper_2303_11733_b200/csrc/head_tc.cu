// K5/K6 on the 5th-generation tensor cores — the whole FC head of a training step
// (fc1 -> fc2 -> fc3 -> Huber -> fc3/fc2/fc1 backward, gnn.py:265-299, numerics.py:58-73) in ONE
// launch of ONE thread-block cluster of 8 CTAs, for the configs[1] head (G <= 256 graphs,
// hidden 512, u width 576, bf16).  Opt-in (dippm_head_tc_enable(1) / DIPPM_HEAD_TC=1): measured
// at ~130 us per head against ~35 us for the 148-CTA mma.sync kernel (head_fused.cu), which stays
// the default -- on 8 SMs the A-operand streaming runs at ~33 GB/s per SM (one 16 KB box per
// ~0.5 us) and the dropout-hash epilogues and row reductions that the mma.sync kernel spreads
// over every SM take ~5-10 us per phase (profiles/r2_head_tc_trace.txt).  Kept as the tested
// tcgen05 / TMA / TMEM formulation of the head (tests/test_gpu_head_tc.py).
//
// CTA c of the cluster owns output columns [64c, 64c + 64) of every hidden-width product.
// Six tensor-core passes, each M = the graphs (two 128-row tiles) or the weight rows, N = 64,
// fp32 accumulators in TMEM: one thread streams the pass's A operand through a 6-stage ring
// (TMA, 128B swizzle, 128 x 64 bf16 boxes) and issues tcgen05.mma (kind::f16, M = 128, N = 64,
// K = 16) against the CTA's B slice (loaded once per pass by TMA); the 4 warps then drain the
// accumulators (tcgen05.ld) through the fused epilogue.  Cluster barriers separate the
// passes whose A operand another CTA produced (its stores are fenced for the async proxy).
//
//   P1  x2[:, c] = drop(relu(u @ W1[:, c] + b1))      A = u (K-major),  B = W1 cols (MN-major)
//   P2  x3[:, c] = drop(relu(x2 @ W2[:, c] + b2))     A = x2,          B = W2 cols;  + fc3 partials
//   C   fc3 (partials summed in CTA order), de-normalise-free Huber terms, dout   (CUDA cores)
//   D   d2[:, c] = (dout W3^T) [x3 > 0] keep, db2, dW3 rows c; loss, db3          (CUDA cores)
//   P3  d1[:, c] = (d2 @ W2^T[:, c]) [x2 > 0] keep    A = d2,          B = W2 rows c (K-major)
//   P4  dW2[:, c] = x2^T @ d2[:, c]                   A = x2 (MN-major), B = d2 cols (MN-major)
//   E   db1                                                                       (CUDA cores)
//   P5  du[:, c] = d1 @ W1[:hp]^T[:, c]               A = d1,          B = W1 rows c (K-major)
//   P6  dW1[:, c] = u^T @ d1[:, c]                    A = u (MN-major), B = d1 cols (MN-major)
//
// Every reduction has a fixed order (deterministic).  Dropout draws use the counter hash and
// index of the GEMM epilogue (tc_gemm.cu) and the mma.sync head, so all three draw the same masks.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace dippm {
namespace tc {
int make_map_sw128(CUtensorMap* map, const dippm_act_t& v, int64_t rows, int64_t cols, int box_cols, int box_rows);
}

namespace htc {

constexpr int kCluster = 8;      // CTAs; each owns 64 of the 512 hidden columns
constexpr int kThreads = 256;    // 8 warps: TMEM lane quarter = warp % 4, column half = warp / 4
constexpr int kHp = 512, kUw = 576, kMaxG = 256;
constexpr int kN = 64;           // output columns per CTA (MMA N)
constexpr int kStages = 8;
constexpr int kATile = 128 * 128;  // 128 rows x 64 bf16 (one K-major box, or two 64 x 64 MN-major boxes)
constexpr int kBMax = 9 * 8192;    // B slice: up to 9 k-blocks of 64 x 64 bf16
constexpr int kSmem = kStages * kATile + kBMax + 1024 + 8192;  // + barriers, bit masks, reduction scratch

// diagnostics: CTA 0's globaltimer at kernel start and after each phase (dippm_head_tc_trace)
__device__ unsigned long long g_trace[16];
#define HTC_STAMP(i) \
  if (blockIdx.x == 0 && threadIdx.x == 0) g_trace[i] = gtime()

struct Maps {  // 128B-swizzled tensor maps (see the launcher)
  CUtensorMap u_k, u_mn, x2_k, x2_mn, d2_k, d2_mn, d1_k, d1_mn, w1, w2;
};

struct Args {
  int G;
  const float *b1, *b2, *w3, *b3;
  __nv_bfloat16 *x2, *x3, *d2, *d1;
  float *d2f, *d1f;
  uint32_t* bits;
  int64_t bits_ld;
  int drop_mode;
  float drop_p, keep_scale;
  uint64_t seed1, seed2;
  const int64_t* seed_dev;
  float* out;
  const double* norm;
  const double* y_raw;
  double delta, grad_den;
  double* loss_out;
  double* row_loss;
  float* dout;
  float *gw1, *gb1, *gw2, *gb2, *gw3, *gb3, *du;
  float* part;  // fc3 partials [16][G][3] (scratch: the du buffer, written last)
  long long* step_counter;
};

// ---- PTX shims ------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0, spins = 0;
  uint64_t t0 = 0;
  while (true) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(su32(b)), "r"(parity)
        : "memory");
    if (done) return;
    if (++spins == 64) t0 = gtime();
    if (spins > 64 && (spins & 255) == 0 && gtime() - t0 > 2000000000ull) __trap();  // protocol bug: fail loudly
  }
}
__device__ __forceinline__ void tma_load(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
          "r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(su32(bar)), "r"(x), "r"(y), "r"(0)
      : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// UMMA shared-memory descriptor: start >> 4, LBO >> 4 at 16, SBO >> 4 at 32, version 1, 128B swizzle
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}
// kind::f16 instruction descriptor: fp32 D, bf16 A/B, A/B MN-major bits, N >> 3, M >> 4
__host__ __device__ constexpr uint32_t idesc(bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(kN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// this CTA's global stores before the barrier are seen by the other CTAs' TMA (async proxy) reads after it
__device__ __forceinline__ void publish_and_sync() {
  __threadfence();
  asm volatile("fence.proxy.async.global;" ::: "memory");
  cluster_sync();
}

// ---- one tensor-core pass ------------------------------------------------------------------------
struct Pass {
  const CUtensorMap* ma;  // A: K-major (box 64 k x 128 rows) or MN-major (box 64 m x 64 k)
  bool a_mn;
  const CUtensorMap* mb;  // B: this CTA's 64-wide slice, per k-block one 64 x 64 box
  bool b_mn;
  int b_x, b_y_step;      // B box of k-block kb at (x, y) = K-major: (kb * 64, b_x) / MN-major: (b_x, kb * 64)
  int m_tiles, kblocks;
};

struct Pipe {  // ring / barrier phase state, carried across passes (single issuing thread)
  uint32_t load_it, mma_it, bphase, dphase;
};

// Thread 0 issues every TMA and MMA of the pass; the accumulator of M-tile mt is TMEM columns
// [mt * 64, mt * 64 + 64).  On return (all threads) the accumulators are complete.
__device__ void run_pass(const Pass& P, uint8_t* ring, uint8_t* bslice, uint64_t* full, uint64_t* empty,
                         uint64_t* bbar, uint64_t* dbar, uint32_t tbase, Pipe& pp) {
  if (threadIdx.x == 0) {
    // B slice once
    mbar_expect(bbar, P.kblocks * 8192);
    for (int kb = 0; kb < P.kblocks; ++kb) {
      if (P.b_mn) tma_load(bslice + kb * 8192, P.mb, bbar, P.b_x, kb * 64);
      else tma_load(bslice + kb * 8192, P.mb, bbar, kb * 64, P.b_x);
    }
    const int items = P.m_tiles * P.kblocks;
    auto load = [&](int j) {
      const uint32_t it = pp.load_it++;
      const int s = it % kStages;
      if (it >= (uint32_t)kStages) mbar_wait(&empty[s], ((it / kStages) - 1) & 1);
      mbar_expect(&full[s], kATile);
      const int mt = j / P.kblocks, kb = j % P.kblocks;
      uint8_t* dst = ring + s * kATile;
      if (!P.a_mn) {
        tma_load(dst, P.ma, &full[s], kb * 64, mt * 128);
      } else {
        tma_load(dst, P.ma, &full[s], mt * 128, kb * 64);
        tma_load(dst + 8192, P.ma, &full[s], mt * 128 + 64, kb * 64);
      }
    };
    // loads run kStages - 2 items ahead: refilling a stage waits for the MMAs two items back,
    // so the previous item's MMAs are still queued on the tensor pipe when this item's issue
    constexpr int kAhead = kStages - 2;
    const int pre = items < kAhead ? items : kAhead;
    for (int j = 0; j < pre; ++j) load(j);
    mbar_wait(bbar, pp.bphase & 1);
    ++pp.bphase;
    fence_after();
    const uint32_t id = idesc(P.a_mn, P.b_mn);
    for (int i = 0; i < items; ++i) {
      const uint32_t it = pp.mma_it++;
      const int s = it % kStages;
      mbar_wait(&full[s], (it / kStages) & 1);
      fence_after();
      const int mt = i / P.kblocks, kb = i % P.kblocks;
      const uint32_t sa = su32(ring + s * kATile), sb = su32(bslice + kb * 8192);
#pragma unroll
      for (int j = 0; j < 4; ++j) {  // K = 16 per MMA
        const uint64_t a = P.a_mn ? sdesc(sa + j * 2048, 8192, 1024) : sdesc(sa + j * 32, 16, 1024);
        const uint64_t b = P.b_mn ? sdesc(sb + j * 2048, 8192, 1024) : sdesc(sb + j * 32, 16, 1024);
        mma(tbase + mt * kN, a, b, id, (kb > 0 || j > 0) ? 1u : 0u);
      }
      commit(&empty[s]);
      if (i + kAhead < items) load(i + kAhead);
    }
    commit(dbar);
  }
  __syncwarp();
  // everyone waits for the accumulators (a single waiter per warp, then the warp)
  if ((threadIdx.x & 31) == 0) mbar_wait(dbar, pp.dphase & 1);
  __syncwarp();
  ++pp.dphase;
  fence_after();
}

// this thread's accumulator row (TMEM lane 32 (warp % 4) + lane) of M-tile mt, the 32 fp32
// columns of its warp's half (warp / 4)
__device__ __forceinline__ int epi_row() { return ((threadIdx.x >> 5) & 3) * 32 + (threadIdx.x & 31); }
__device__ __forceinline__ int epi_half() { return threadIdx.x >> 7; }
__device__ __forceinline__ void acc_row(uint32_t tbase, int mt, float (&v)[32]) {
  const uint32_t lane_base = (uint32_t)(((threadIdx.x >> 5) & 3) * 32) << 16;
  uint32_t r[32];
  tmem_ld32(tbase + lane_base + mt * kN + epi_half() * 32, r);
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void store_bf16_32(__nv_bfloat16* dst, const float (&v)[32]) {
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    __nv_bfloat162 h[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[q * 8 + 2 * i], v[q * 8 + 2 * i + 1]);
    d[q] = *reinterpret_cast<uint4*>(h);
  }
}

__global__ void __cluster_dims__(kCluster, 1, 1) __launch_bounds__(kThreads, 1)
    k_head_tc(const __grid_constant__ Maps M, Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;
  uint8_t* bslice = ring + kStages * kATile;
  uint64_t* full = reinterpret_cast<uint64_t*>(bslice + kBMax);
  uint64_t* empty = full + kStages;
  uint64_t* bbar = empty + kStages;
  uint64_t* dbar = bbar + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(dbar + 1);
  uint32_t* s_x2b = tslot + 4;          // [256][2] x2 > 0 bits of this CTA's columns (P1 -> P3)
  uint32_t* s_x3b = s_x2b + 2 * kMaxG;  // [256][2] x3 > 0 bits (P2 -> D)
  double* s_red = reinterpret_cast<double*>(s_x3b + 2 * kMaxG);  // [8]
  const int c = (int)cluster_rank();
  const int col0 = c * kN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.G, mtiles = (G + 127) / 128;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(bbar, 1);
    mbar_init(dbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = *tslot;
  Pipe pp{0, 0, 0, 0};
  const float keep = 1.0f / (1.0f - a.drop_p);
  auto drop_seed = [&](uint64_t s) {
    return (a.drop_mode == 2 && a.seed_dev) ? s ^ ((uint64_t)a.seed_dev[0] * 0x9E3779B97F4A7C15ull) : s;
  };

  HTC_STAMP(0);
  // ---- P1: x2 = drop(relu(u W1 + b1)) (+ bit masks) -------------------------------------------
  const int hc = epi_half(), cc = col0 + 32 * hc;  // this warp's 32 columns
  run_pass(Pass{&M.u_k, false, &M.w1, true, col0, 0, mtiles, kUw / 64}, ring, bslice, full, empty, bbar, dbar, tbase,
           pp);
  {
    const uint64_t seed = drop_seed(a.seed1);
    for (int mt = 0; mt < mtiles; ++mt) {
      const int row = mt * 128 + epi_row();
      float v[32];
      acc_row(tbase, mt, v);
      uint32_t bw = 0u;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        float x = fmaxf(v[j] + __ldg(a.b1 + cc + j), 0.f);
        if (a.drop_mode == 2) x *= uniform_hash(seed, (uint64_t)((int64_t)row * kHp + cc + j)) >= a.drop_p ? keep : 0.f;
        v[j] = x;
        bw |= (uint32_t)(x > 0.f) << j;
      }
      if (row < G) {
        store_bf16_32(a.x2 + (int64_t)row * kHp + cc, v);
        a.bits[(int64_t)(2 * c + hc) * a.bits_ld + row] = bw;
        s_x2b[row * 2 + hc] = bw;
      }
    }
  }
  fence_before();
  publish_and_sync();
  fence_after();

  HTC_STAMP(1);
  // ---- P2: x3 = drop(relu(x2 W2 + b2)), fc3 partials over this warp's 32 columns ------------------
  __nv_bfloat16* x3s = reinterpret_cast<__nv_bfloat16*>(ring);  // [256][64] this CTA's x3 (for D)
  run_pass(Pass{&M.x2_k, false, &M.w2, true, col0, 0, mtiles, kHp / 64}, ring, bslice, full, empty, bbar, dbar, tbase,
           pp);
  {
    const uint64_t seed = drop_seed(a.seed2);
    for (int mt = 0; mt < mtiles; ++mt) {
      const int row = mt * 128 + epi_row();
      float v[32];
      acc_row(tbase, mt, v);
      uint32_t bw = 0u;
      float p0 = 0.f, p1 = 0.f, p2 = 0.f;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        float x = fmaxf(v[j] + __ldg(a.b2 + cc + j), 0.f);
        if (a.drop_mode == 2) x *= uniform_hash(seed, (uint64_t)((int64_t)row * kHp + cc + j)) >= a.drop_p ? keep : 0.f;
        const float xb = __bfloat162float(__float2bfloat16_rn(x));  // fc3 and dW3 read the stored bf16 x3
        v[j] = x;
        bw |= (uint32_t)(x > 0.f) << j;
        p0 = fmaf(xb, __ldg(a.w3 + (cc + j) * 3 + 0), p0);
        p1 = fmaf(xb, __ldg(a.w3 + (cc + j) * 3 + 1), p1);
        p2 = fmaf(xb, __ldg(a.w3 + (cc + j) * 3 + 2), p2);
      }
      if (row < G) {
        store_bf16_32(a.x3 + (int64_t)row * kHp + cc, v);
        store_bf16_32(x3s + row * kN + 32 * hc, v);
        s_x3b[row * 2 + hc] = bw;
        float* pr = a.part + ((int64_t)(2 * c + hc) * G + row) * 3;
        pr[0] = p0;
        pr[1] = p1;
        pr[2] = p2;
      }
    }
  }
  publish_and_sync();

  HTC_STAMP(2);
  // ---- C: fc3 + Huber terms (CTA c: graphs [32c, 32c + 32), 4 lanes per graph, k = lane % 4) ----
  if (threadIdx.x < 128) {
    const int g = 32 * c + (threadIdx.x >> 2), k = threadIdx.x & 3;
    const bool ok = g < G && k < 3;
    double le_k = 0.0;
    if (ok) {
      float pq[2 * kCluster];
#pragma unroll
      for (int q = 0; q < 2 * kCluster; ++q) pq[q] = __ldcg(a.part + ((int64_t)q * G + g) * 3 + k);
      float sp = 0.f;
#pragma unroll
      for (int q = 0; q < 2 * kCluster; ++q) sp += pq[q];  // column-slice order
      const float o = __ldg(a.b3 + k) + sp;
      a.out[g * 3 + k] = o;
      const double pred = (double)o, y = a.y_raw[g * 3 + k];  // k_huber's per-graph terms (head.cu)
      const double t = (y - a.norm[k]) / a.norm[3 + k];
      const double r = pred - t, ab = fabs(r);
      const bool quad = ab <= a.delta;
      le_k = quad ? 0.5 * r * r : a.delta * (ab - 0.5 * a.delta);
      const double gr = quad ? r : a.delta * (r > 0 ? 1.0 : (r < 0 ? -1.0 : 0.0));
      a.dout[g * 3 + k] = (float)(gr / 3.0 / a.grad_den);
      const double den = pred * a.norm[3 + k] + a.norm[k];
      a.row_loss[(int64_t)g * 4 + 1 + k] = fabs(den - y) / fabs(y);
    }
    const double l1 = __shfl_down_sync(0xffffffffu, le_k, 1, 4), l2 = __shfl_down_sync(0xffffffffu, le_k, 2, 4);
    if (k == 0 && g < G) a.row_loss[(int64_t)g * 4] = ((0.0 + le_k) + l1 + l2) / 3.0;
  }
  publish_and_sync();

  HTC_STAMP(3);
  // ---- D: d2 = (dout W3^T) [x3 > 0] keep (this CTA's columns), db2, dW3 rows; loss + db3 (CTA 0) ----
  {
    float* dout_s = reinterpret_cast<float*>(ring + 32768);  // [256][3]
    for (int i = threadIdx.x; i < 3 * G; i += kThreads) dout_s[i] = __ldcg(a.dout + i);
    __syncthreads();
    const int j = threadIdx.x & 63, rg = threadIdx.x >> 6;  // column, row group (g = rg mod 4)
    const int col = col0 + j;
    const float w0 = __ldg(a.w3 + col * 3), w1 = __ldg(a.w3 + col * 3 + 1), w2 = __ldg(a.w3 + col * 3 + 2);
    float cb = 0.f, s0 = 0.f, s1 = 0.f, s2 = 0.f;
    for (int g = rg; g < G; g += 4) {
      const float e0 = dout_s[g * 3], e1 = dout_s[g * 3 + 1], e2 = dout_s[g * 3 + 2];
      const float dx = e0 * w0 + e1 * w1 + e2 * w2;
      const bool pos = (s_x3b[g * 2 + (j >> 5)] >> (j & 31)) & 1u;
      const float dv = pos ? dx * a.keep_scale : 0.f;
      a.d2[(int64_t)g * kHp + col] = __float2bfloat16_rn(dv);
      a.d2f[(int64_t)g * kHp + col] = dv;
      cb += dv;
      const float x = __bfloat162float(x3s[g * kN + j]);
      s0 = fmaf(x, e0, s0);
      s1 = fmaf(x, e1, s1);
      s2 = fmaf(x, e2, s2);
    }
    float* sf = reinterpret_cast<float*>(ring + 36864);  // [4][64][4]: the row groups, added in order
    sf[(rg * 64 + j) * 4 + 0] = cb;
    sf[(rg * 64 + j) * 4 + 1] = s0;
    sf[(rg * 64 + j) * 4 + 2] = s1;
    sf[(rg * 64 + j) * 4 + 3] = s2;
    __syncthreads();
    if (rg == 0) {
      float t[4];
      for (int k = 0; k < 4; ++k)
        t[k] = ((sf[j * 4 + k] + sf[(64 + j) * 4 + k]) + sf[(128 + j) * 4 + k]) + sf[(192 + j) * 4 + k];
      a.gb2[col] = t[0];
      for (int k = 0; k < 3; ++k) a.gw3[col * 3 + k] = t[1 + k];
    }
    if (c == 0) {  // batch loss (fixed order: per-thread strided sums, xor tree, warps in order) and db3
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      float b[3] = {0.f, 0.f, 0.f};
      for (int g = threadIdx.x; g < G; g += kThreads) {
        for (int k = 0; k < 4; ++k) acc[k] += __ldcg(a.row_loss + (int64_t)g * 4 + k);
        for (int k = 0; k < 3; ++k) b[k] += dout_s[g * 3 + k];
      }
      double t[4];
      float tb[3];
      for (int k = 0; k < 4; ++k) {
        double v = acc[k];
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        __syncthreads();
        if (lane == 0) s_red[warp] = v;
        __syncthreads();
        double tt = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) tt += s_red[w];
        t[k] = tt;
      }
      for (int k = 0; k < 3; ++k) {
        float v = b[k];
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        __syncthreads();
        if (lane == 0) reinterpret_cast<float*>(s_red)[warp] = v;
        __syncthreads();
        float tt = 0.f;
        for (int w = 0; w < kThreads / 32; ++w) tt += reinterpret_cast<float*>(s_red)[w];
        tb[k] = tt;
      }
      if (threadIdx.x == 0) {
        a.loss_out[0] = t[0] / (double)G;
        for (int k = 0; k < 3; ++k) a.loss_out[1 + k] = t[1 + k];
        for (int k = 0; k < 3; ++k) a.gb3[k] = tb[k];
      }
    }
  }
  fence_before();
  publish_and_sync();
  fence_after();

  HTC_STAMP(4);
  // ---- P3: d1 = (d2 W2^T) [x2 > 0] keep; db1 from the rows staged in shared memory -----------------
  run_pass(Pass{&M.d2_k, false, &M.w2, false, col0, 0, mtiles, kHp / 64}, ring, bslice, full, empty, bbar, dbar, tbase,
           pp);
  {
    float* d1s = reinterpret_cast<float*>(ring);  // [256][64] (the ring is idle until P4)
    for (int mt = 0; mt < mtiles; ++mt) {
      const int row = mt * 128 + epi_row();
      float v[32];
      acc_row(tbase, mt, v);
      const uint32_t bw = row < G ? s_x2b[row * 2 + hc] : 0u;
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = (bw >> j) & 1u ? v[j] * a.keep_scale : 0.f;
      if (row < G) {
        store_bf16_32(a.d1 + (int64_t)row * kHp + cc, v);
        float4* df = reinterpret_cast<float4*>(a.d1f + (int64_t)row * kHp + cc);
        float4* ds = reinterpret_cast<float4*>(d1s + row * kN + 32 * hc);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 f = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          df[q] = f;
          ds[q] = f;
        }
      }
    }
    __syncthreads();
    const int j = threadIdx.x & 63, rg = threadIdx.x >> 6;
    float cb = 0.f;
    for (int g = rg; g < G; g += 4) cb += d1s[g * kN + j];
    float* sf = reinterpret_cast<float*>(ring + 65536);  // [4][64]
    sf[rg * 64 + j] = cb;
    __syncthreads();
    if (rg == 0) a.gb1[col0 + j] = ((sf[j] + sf[64 + j]) + sf[128 + j]) + sf[192 + j];
  }
  fence_before();
  __syncthreads();
  fence_after();

  HTC_STAMP(5);
  // ---- P4: dW2[:, c] = x2^T d2[:, c] (M = 512 in 4 tiles, K = G) ----------------------------------
  const int gk = (G + 63) / 64;
  run_pass(Pass{&M.x2_mn, true, &M.d2_mn, true, col0, 0, kHp / 128, gk}, ring, bslice, full, empty, bbar, dbar, tbase,
           pp);
  for (int mt = 0; mt < kHp / 128; ++mt) {
    const int m = mt * 128 + epi_row();
    float v[32];
    acc_row(tbase, mt, v);
    float4* gw = reinterpret_cast<float4*>(a.gw2 + (int64_t)m * kHp + cc);
#pragma unroll
    for (int q = 0; q < 8; ++q) gw[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  }
  fence_before();
  publish_and_sync();  // d1 complete on every CTA
  fence_after();

  HTC_STAMP(6);
  // ---- P5: du[:, c] = d1 W1[:hp]^T[:, c] (the readout gradient) ----------------------------------------
  run_pass(Pass{&M.d1_k, false, &M.w1, false, col0, 0, mtiles, kHp / 64}, ring, bslice, full, empty, bbar, dbar, tbase,
           pp);
  for (int mt = 0; mt < mtiles; ++mt) {
    const int row = mt * 128 + epi_row();
    float v[32];
    acc_row(tbase, mt, v);
    if (row < G) {
      float4* d = reinterpret_cast<float4*>(a.du + (int64_t)row * kHp + cc);
#pragma unroll
      for (int q = 0; q < 8; ++q) d[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
  }
  fence_before();
  __syncthreads();
  fence_after();

  HTC_STAMP(7);
  // ---- P6: dW1[:, c] = u^T d1[:, c] (M = 576 in 5 tiles, K = G) ----------------------------------
  run_pass(Pass{&M.u_mn, true, &M.d1_mn, true, col0, 0, (kUw + 127) / 128, gk}, ring, bslice, full, empty, bbar, dbar,
           tbase, pp);
  for (int mt = 0; mt < (kUw + 127) / 128; ++mt) {
    const int m = mt * 128 + epi_row();
    float v[32];
    acc_row(tbase, mt, v);
    if (m < kUw) {
      float4* gw = reinterpret_cast<float4*>(a.gw1 + (int64_t)m * kHp + cc);
#pragma unroll
      for (int q = 0; q < 8; ++q) gw[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
  }
  HTC_STAMP(8);
  // the dropout draws (which read the step counter) are all done: advance it for Adam
  if (c == 0 && threadIdx.x == 0 && a.step_counter) a.step_counter[0] += 1;
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
}

}  // namespace htc

int head_tc_trace(unsigned long long* out16) {
  return cudaMemcpyFromSymbol(out16, htc::g_trace, sizeof(htc::g_trace)) == cudaSuccess ? 0 : 2;
}

// Launch the tensor-core head when the batch fits it (returns false to fall back).
bool head_tc_launch(const dippm_head_args_t* h, cudaStream_t s, int32_t* status) {
  using namespace htc;
  if (!(h->G >= 1 && h->G <= kMaxG && h->hp == kHp && h->u_width == kUw && h->train && h->y_raw && h->du &&
        h->gw1 && h->gw2 &&
        h->drop_mode != 1 && !h->pool_partial && !h->y_pred && h->bits && h->bits_ld >= h->G))
    return false;
  *status = DIPPM_OK;
  auto fail = [&](int32_t st) {
    *status = st;
    return true;
  };
  const int G = (int)h->G;
  auto act = [](const void* p, int64_t ld) { return dippm_act_t{const_cast<void*>(p), ld, 0, DIPPM_DT_BF16}; };
  Maps M;
  int st = 0;
  st |= tc::make_map_sw128(&M.u_k, act(h->u, kUw), G, kUw, 64, 128);
  st |= tc::make_map_sw128(&M.u_mn, act(h->u, kUw), G, kUw, 64, 64);
  st |= tc::make_map_sw128(&M.x2_k, act(h->x2, kHp), G, kHp, 64, 128);
  st |= tc::make_map_sw128(&M.x2_mn, act(h->x2, kHp), G, kHp, 64, 64);
  st |= tc::make_map_sw128(&M.d2_k, act(h->d2, kHp), G, kHp, 64, 128);
  st |= tc::make_map_sw128(&M.d2_mn, act(h->d2, kHp), G, kHp, 64, 64);
  st |= tc::make_map_sw128(&M.d1_k, act(h->d1, kHp), G, kHp, 64, 128);
  st |= tc::make_map_sw128(&M.d1_mn, act(h->d1, kHp), G, kHp, 64, 64);
  st |= tc::make_map_sw128(&M.w1, act(h->w1, kHp), kUw, kHp, 64, 64);
  st |= tc::make_map_sw128(&M.w2, act(h->w2, kHp), kHp, kHp, 64, 64);
  if (st) return fail(DIPPM_ERR_ARG);
  Args a{};
  a.G = G;
  a.b1 = h->b1;
  a.b2 = h->b2;
  a.w3 = h->w3;
  a.b3 = h->b3;
  a.x2 = reinterpret_cast<__nv_bfloat16*>(h->x2);
  a.x3 = reinterpret_cast<__nv_bfloat16*>(h->x3);
  a.d2 = reinterpret_cast<__nv_bfloat16*>(h->d2);
  a.d1 = reinterpret_cast<__nv_bfloat16*>(h->d1);
  a.d2f = h->d2f;
  a.d1f = h->d1f;
  a.bits = h->bits;
  a.bits_ld = h->bits_ld;
  a.drop_mode = h->drop_mode;
  a.drop_p = (float)h->drop_p;
  a.keep_scale = h->keep_scale;
  a.seed1 = h->seed1;
  a.seed2 = h->seed2;
  a.seed_dev = h->seed_dev;
  a.out = h->out;
  a.norm = h->norm;
  a.y_raw = h->y_raw;
  a.delta = h->delta;
  a.grad_den = h->grad_den > 0 ? h->grad_den : (double)G;
  a.loss_out = h->loss_out;
  a.row_loss = h->row_loss;
  a.dout = h->dout;
  a.gw1 = h->gw1;
  a.gb1 = h->gb1;
  a.gw2 = h->gw2;
  a.gb2 = h->gb2;
  a.gw3 = h->gw3;
  a.gb3 = h->gb3;
  a.du = h->du;
  a.part = h->du;  // fc3 partials [8][G][3] live in du until P5 overwrites it
  a.step_counter = reinterpret_cast<long long*>(h->step_counter);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_head_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return fail(cuda_status(e, "head_tc attribute"));
    attr = true;
  }
  k_head_tc<<<kCluster, kThreads, kSmem, s>>>(M, a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(cuda_status(e, "k_head_tc"));
  count_launches(1);
  return true;
}

}  // namespace dippm
