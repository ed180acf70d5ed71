// K3 — SAGE projections and their gradients on the 5th-generation tensor cores.
//
//   FWD   z = [h | m] @ [W_self; W_neigh] + b, h' = relu(z)     gnn.py:207-209
//   STORE dA = dz @ [W_self; W_neigh]^T                           gnn.py:232
//   WGRAD dW = [h | m]^T @ dz (split over node-row chunks)        gnn.py:228-229
//
// One persistent kernel template, warp-specialised (192 threads, 1 CTA/SM):
//   warp 0      TMA producer: 3-D tensor maps (cols, rows, plane) with 128B
//               swizzle feed a kStages-deep shared-memory ring (mbarriers);
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer; the fp32
//               accumulator (128 x BN) lives in TMEM, double-buffered so the
//               epilogue of tile i overlaps the MMAs of tile i+1;
//   warps 2-9   epilogue (two warps per TMEM lane quarter, alternate 32-column
//               chunks): tcgen05.ld (32x32b.x32) -> bias/ReLU/gate -> smem -> TMA store.
// Operand precision:
//   bf16  kind::f16, one pass;
//   tf32x3 kind::tf32 on hi/lo planes, 3 passes (hi*hi + hi*lo + lo*hi) so
//          products carry ~22 mantissa bits: fp32-grade results on tensor cores.
// Operand majorness: K-major for FWD/STORE; both MN-major for WGRAD (dz and
// [h|m] are row-major [nodes, features] and the reduction runs over nodes),
// which the UMMA descriptors express directly (no transposed copies).
#include <cstdlib>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace dippm {
namespace tc {

constexpr int kThreads = 64 + 256;  // TMA warp, MMA warp, 8 epilogue warps
constexpr int kBM = 128;
enum { EPI_FWD = 0, EPI_STORE = 1, EPI_PARTIAL = 2, EPI_GATE = 3, EPI_FWD_DROP = 4 };

struct Params {
  int64_t M, N, K;
  int splits;
  int m_tiles, n_tiles;
  const float* bias;
  int relu;
  ActView out;
  float* c;
  int64_t ldc;
  ActView gate;      // EPI_GATE: out = gate > 0 ? acc * gate_scale : 0
  float gate_scale;
  int drop_mode;     // EPI_FWD dropout: 0 none, 1 multiply mask[], 2 generate into mask[]
  float* mask;
  int64_t ldm;
  float drop_p;
  uint64_t seed;
  const int64_t* seed_dev;
  uint32_t* relu_bits;        // FWD: optional 1-bit (out > 0) mask, word [(c/32)*bits_ld + r] (chunk-major)
  const uint32_t* gate_bits;  // GATE: optional 1-bit gate instead of gate values
  int64_t bits_ld;
  // WGRAD output: reduce_mode 0 = partials to c only; 1 = fused reduce, every split CTA
  // reduces a row slice once all splits of its tile have landed (all tiles co-resident);
  // 2 = fused reduce by the last split to arrive; 3 = single split, write wout directly.
  int reduce_mode;
  float* wout;
  int64_t ldo;
  double out_scale;
  int* sync;
  // FWD with the fused readout (pool != nullptr): segmented column sums per 32-row block
  float* pool_part;
  float* pool_graph;
  const int* node_graph;
  const int* graph_ptr;
  const float* bias_part;  // WGRAD (optional): fold these partial rows of the layer's bias gradient
  const int* bias_count;   //   (their count, written by the producing aggregation kernel)
  float* bias_fold;        //   into this [N] fp32 vector (column sums in row order, fp64)
  unsigned long long* ts;  // diagnostics only (DIPPM_GEMM_TS=<device address>): per-CTA globaltimer stamps
  int dbg;  // diagnostics only (DIPPM_GEMM_DEBUG): bit 0 skip epilogue stores, bit 1 skip the
            // bit masks, bit 2 skip the whole chunk loop (release the accumulator at once), bit 3
            // use the per-float FWD epilogue instead of the packed one (1-CTA tiles)
};

// ------------------------------------------------------------------ PTX shims
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Bounded wait: a protocol bug traps (launch error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  uint32_t spins = 0;
  uint64_t t0 = 0;
  while (true) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
    if (done) return;
    ++spins;
    if (spins == 64) t0 = globaltimer();
    if (spins > 64 && (spins & 255) == 0 && globaltimer() - t0 > 2000000000ull) __trap();
  }
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

template <int kFmt>
__device__ __forceinline__ void umma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (kFmt == 1) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  }
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// Issue only (no wait): the registers are valid after the next tmem_wait_ld().
__device__ __forceinline__ void tmem_ld32_issue(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
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

// Shared-memory matrix descriptor (sm_100 UMMA): start>>4 [0,14), LBO>>4
// [16,30), SBO>>4 [32,46), version 1 at bit 46, swizzle mode 2 (128B) [61,64).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint64_t layout = 2) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (layout << 61);
}
// Instruction descriptor, kind::f16 / kind::tf32: D fp32 [4,6), A/B format
// [7,10)/[10,13) (1 = bf16, 2 = tf32), A/B MN-major bits 15/16, N>>3 [17,23),
// M>>4 [24,29).
__host__ __device__ constexpr uint32_t make_idesc(int fmt, bool a_mn, bool b_mn, int M, int N) {
  return (1u << 4) | ((uint32_t)fmt << 7) | ((uint32_t)fmt << 10) | ((a_mn ? 1u : 0u) << 15) |
         ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// GATE epilogue helpers: 32 gate values (the layer-below activation, in the
// GEMM's operand dtype) -> a 32-bit (gate > 0) mask.  Loads are issued one
// chunk ahead and decoded after the next chunk's math (latency hiding).
// tf32x3: the sign of v = hi + lo is the sign of hi unless hi == 0 (|v| below
// the tf32 grid, essentially exact zeros), where the lo plane decides.
template <int kFmt>
__device__ __forceinline__ void gate_issue(const ActView& g, int64_t row, int n, uint4 (&r)[8]) {
  if constexpr (kFmt == 1) {
    const uint4* p = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(g.base) + row * g.ld + n);
#pragma unroll
    for (int i = 0; i < 4; ++i) r[i] = __ldg(p + i);
  } else {
    const uint4* p = reinterpret_cast<const uint4*>(reinterpret_cast<const float*>(g.base) + row * g.ld + n);
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = __ldg(p + i);
  }
}
template <int kFmt>
__device__ __forceinline__ uint32_t gate_mask(const ActView& g, int64_t row, int n, const uint4 (&r)[8]) {
  uint32_t m = 0;
  if constexpr (kFmt == 1) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t w[4] = {r[i].x, r[i].y, r[i].z, r[i].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t lo = w[j] & 0xFFFFu, hi = w[j] >> 16;  // bf16 > 0: sign clear, not zero
        m |= (uint32_t)(!(lo & 0x8000u) && (lo & 0x7FFFu)) << (i * 8 + j * 2);
        m |= (uint32_t)(!(hi & 0x8000u) && (hi & 0x7FFFu)) << (i * 8 + j * 2 + 1);
      }
    }
  } else {
    const float* lo_plane = reinterpret_cast<const float*>(g.base) + g.plane_stride + row * g.ld + n;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t w[4] = {r[i].x, r[i].y, r[i].z, r[i].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        bool pos = (int32_t)w[j] > 0;
        if (w[j] == 0u || w[j] == 0x80000000u) pos = lo_plane[i * 4 + j] > 0.f;
        m |= (uint32_t)pos << (i * 4 + j);
      }
    }
  }
  return m;
}

// Activation-writing epilogues stage each warp's 32 rows x 32 columns in shared
// memory and hand them to the TMA engine (cp.async.bulk.tensor store): fully
// coalesced, asynchronous, and rows beyond M are clipped by the tensor map.
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int x, int y, int z) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(x), "r"(y), "r"(z)
               : "memory");
}

// Each of the 8 epilogue warps owns 4 KB of staging: two 2 KB slots for bf16
// output (one TMA store stays in flight while the next chunk is computed), one
// slot for fp32, and for tf32 hi/lo the two planes go through the slot in turn.
constexpr int kEpiWarps = 8;
constexpr int kStageWarpBytes = 4096;

__device__ __forceinline__ void stage_wait(int lane, int pending) {
  if (lane == 0) {
    if (pending == 1) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  __syncwarp();
}
__device__ __forceinline__ void stage_issue(const CUtensorMap* map, const uint8_t* stg, int lane, int x, int y, int z) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    tma_store_3d(map, stg, x, y, z);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
}

__device__ __forceinline__ void epi_store_chunk(uint8_t* stg_base, const CUtensorMap* map, int64_t dtype, int lane,
                                                const float (&v)[32], int x, int y, int chunk) {
  if (dtype == DIPPM_DT_BF16) {
    uint8_t* stg = stg_base + (chunk & 1) * 2048;
    stage_wait(lane, 1);  // the slot's previous store has been read
    // 64-byte rows in the TMA 64B-swizzle layout: 16-byte unit k of row r sits at
    // unit k ^ ((r >> 1) & 3), so the 8 lanes of each store phase hit distinct banks.
    uint4* d = reinterpret_cast<uint4*>(stg + lane * 64);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint4 q;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
      for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[k * 8 + 2 * i], v[k * 8 + 2 * i + 1]);
      d[k ^ ((lane >> 1) & 3)] = q;
    }
    stage_issue(map, stg, lane, x, y, 0);
  } else if (dtype == DIPPM_DT_TF32X3) {
    // 128-byte rows in the TMA 128B-swizzle layout: unit k of row r at unit k ^ (r & 7).
    float4* d = reinterpret_cast<float4*>(stg_base + lane * 128);
    float lo[32];
    stage_wait(lane, 0);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float hi[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        hi[i] = tf32_hi(v[4 * k + i]);
        lo[4 * k + i] = tf32_rn(v[4 * k + i] - hi[i]);
      }
      d[k ^ (lane & 7)] = make_float4(hi[0], hi[1], hi[2], hi[3]);
    }
    stage_issue(map, stg_base, lane, x, y, 0);
    stage_wait(lane, 0);
#pragma unroll
    for (int k = 0; k < 8; ++k) d[k ^ (lane & 7)] = make_float4(lo[4 * k], lo[4 * k + 1], lo[4 * k + 2], lo[4 * k + 3]);
    stage_issue(map, stg_base, lane, x, y, 1);
  } else {
    float4* d = reinterpret_cast<float4*>(stg_base + lane * 128);
    stage_wait(lane, 0);
#pragma unroll
    for (int k = 0; k < 8; ++k) d[k ^ (lane & 7)] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
    stage_issue(map, stg_base, lane, x, y, 0);
  }
}

// Packed epilogue helpers (FWD, bf16 output): bias add on the fp32 pair pipe (FADD2), round to
// bf16x2, ReLU on the packed pair (max(round(x), 0) == round(max(x, 0)): rounding is monotone),
// and the 1-bit (stored value > 0) mask from the packed pair (HSETP2) -- about 2.7 instructions per
// element against 5 for the per-float sequence (the layer-1 epilogue is instruction-bound).
__device__ __forceinline__ float2 add_f32x2(float2 a, float2 b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)));
  return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ uint32_t relu_bf16x2(uint32_t w) {
  uint32_t r;
  asm("max.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(w), "r"(0u));
  return r;
}
// bits 2i / 2i+1 of `bits` |= (low / high half of w) > 0
template <int I>
__device__ __forceinline__ void pos_bits_bf16x2(uint32_t& bits, uint32_t w) {
  asm("{\n\t.reg .pred p, q;\n\tsetp.gt.bf16x2 p|q, %1, %2;\n\t@p or.b32 %0, %0, %3;\n\t@q or.b32 %0, %0, %4;\n\t}"
      : "+r"(bits)
      : "r"(w), "r"(0u), "n"(1u << (2 * I)), "n"(1u << (2 * I + 1)));
}
// four independent predicated-OR chains (words i, i+4, i+8, i+12), then a 3-level OR: the
// dependent chain per chunk is 8 ORs instead of 32 (the epilogue runs 2 warps per scheduler)
template <int I>
struct PosBits {
  static __device__ __forceinline__ void run(uint32_t (&b)[4], const uint32_t (&w)[16]) {
    PosBits<I - 1>::run(b, w);
    pos_bits_bf16x2<I - 1>(b[(I - 1) & 3], w[I - 1]);
  }
};
template <>
struct PosBits<0> {
  static __device__ __forceinline__ void run(uint32_t (&)[4], const uint32_t (&)[16]) {}
};
__device__ __forceinline__ uint32_t pos_bits32(const uint32_t (&w)[16]) {
  uint32_t b[4] = {0u, 0u, 0u, 0u};
  PosBits<16>::run(b, w);
  return (b[0] | b[1]) | (b[2] | b[3]);
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ float4 lds128f(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
// 32 packed bf16 of one row (this lane) -> the warp's 64B-swizzled staging slot -> TMA store
__device__ __forceinline__ void epi_store_packed(uint8_t* stg_base, const CUtensorMap* map, int lane,
                                                 const uint32_t (&w)[16], int x, int y, int chunk) {
  uint8_t* stg = stg_base + (chunk & 1) * 2048;
  stage_wait(lane, 1);
  const uint32_t d = smem_u32(stg + lane * 64);
#pragma unroll
  for (int k = 0; k < 4; ++k) sts128(d + ((k ^ ((lane >> 1) & 3)) << 4), w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
  stage_issue(map, stg, lane, x, y, 0);
}

template <int kFmt, int kBN, int kCta>
struct Cfg {
  static constexpr int kElem = kFmt == 1 ? 2 : 4;
  static constexpr int kBK = 128 / kElem;       // one 128-byte swizzle row of K (or of MN) per k-block
  static constexpr int kUK = 32 / kElem;        // K per tcgen05.mma (16 bf16 / 8 tf32)
  static constexpr int kPlanes = kFmt == 1 ? 1 : 2;
  static constexpr int kBNl = kBN / kCta;       // B rows (N) held by each CTA of the pair
  static constexpr int kTileM = kBM * kCta;     // output rows per (cluster) tile
  static constexpr int kATile = kBM * 128;      // bytes per plane
  static constexpr int kBTile = kBNl * 128;
  static constexpr int kStageBytes = kPlanes * (kATile + kBTile);
  // bias staging for the packed FWD epilogue (bf16): up to 1024 columns, paid for by one ring stage
  // fewer on the 1-CTA 256-wide tile (the only shape whose ring fills the shared memory)
  static constexpr int kBiasCols = (kFmt == 1 && kCta == 1 && kBN == 256) ? 1024 : 0;
  static constexpr int kBiasBytes = kBiasCols * 4;
  static constexpr int kRing = 196608 - ((kFmt == 1 && kCta == 1 && kBN == 256) ? kStageBytes : 0);
  static constexpr int kStages = (kRing / kStageBytes) < 8 ? (kRing / kStageBytes) : 8;
  static constexpr int kTmemCols = 2 * kBN;     // double-buffered accumulator
  static constexpr int kEpiStage = kEpiWarps * kStageWarpBytes;  // TMA-store staging of the epilogue warps
  static constexpr int kSmemBytes = kStages * kStageBytes + kEpiStage + kBiasBytes + 1024 + 256;
};

// ---- CTA-pair (cta_group::2) plumbing -------------------------------------
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same shared-memory object in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// TMA load whose completion is signalled on the leader CTA's mbarrier (2-SM mode)
__device__ __forceinline__ void tma_load_3d_pair(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int x, int y,
                                                 int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(x), "r"(y), "r"(z)
      : "memory");
}
template <int kFmt>
__device__ __forceinline__ void umma_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (kFmt == 1) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  }
}
// commit: arrive on the barrier at this offset in both CTAs of the pair once the MMAs retire
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory"); }
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Fixed-order split-K reduction of one CTA's 128-row tile slice: out = scale * sum_s C_s
// (fp64 sums, independent of which CTA reduces, so results are deterministic).  Partials are
// read through L2 (ld.global.cg).  When the slice is small (the layer-1 weight gradient: ~1 row
// x 64 float4 per CTA against 74 splits) the splits are cut into G contiguous groups summed by
// different threads (16 loads in flight each) and the group sums are added in group order in
// shared memory: the reduction is no longer a 74-deep chain of L2 round trips.
template <int kBN>
__device__ __forceinline__ void sum_splits(const Params& p, const float* src, int s0, int s1, double (&a)[4]) {
  const int64_t plane = p.M * p.ldc;
  int s = s0;
  for (; s + 16 <= s1; s += 16) {  // 16 loads in flight, summed in split order
    float4 v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __ldcg(reinterpret_cast<const float4*>(src + (s + j) * plane));
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      a[0] += v[j].x; a[1] += v[j].y; a[2] += v[j].z; a[3] += v[j].w;
    }
  }
  for (; s + 8 <= s1; s += 8) {
    float4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldcg(reinterpret_cast<const float4*>(src + (s + j) * plane));
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      a[0] += v[j].x; a[1] += v[j].y; a[2] += v[j].z; a[3] += v[j].w;
    }
  }
  for (; s + 4 <= s1; s += 4) {
    float4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = __ldcg(reinterpret_cast<const float4*>(src + (s + j) * plane));
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      a[0] += v[j].x; a[1] += v[j].y; a[2] += v[j].z; a[3] += v[j].w;
    }
  }
  for (; s < s1; ++s) {
    const float4 v = __ldcg(reinterpret_cast<const float4*>(src + s * plane));
    a[0] += v.x; a[1] += v.y; a[2] += v.z; a[3] += v.w;
  }
}

// two items at once (twice the loads in flight per round trip), each summed in split order
__device__ __forceinline__ void sum_splits2(const Params& p, const float* src0, const float* src1, int s0, int s1,
                                            double (&a)[4], double (&b)[4]) {
  const int64_t plane = p.M * p.ldc;
  int s = s0;
  for (; s + 8 <= s1; s += 8) {
    float4 v[8], w[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      v[j] = __ldcg(reinterpret_cast<const float4*>(src0 + (s + j) * plane));
      w[j] = __ldcg(reinterpret_cast<const float4*>(src1 + (s + j) * plane));
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      a[0] += v[j].x; a[1] += v[j].y; a[2] += v[j].z; a[3] += v[j].w;
      b[0] += w[j].x; b[1] += w[j].y; b[2] += w[j].z; b[3] += w[j].w;
    }
  }
  for (; s < s1; ++s) {
    const float4 v = __ldcg(reinterpret_cast<const float4*>(src0 + s * plane));
    const float4 w = __ldcg(reinterpret_cast<const float4*>(src1 + s * plane));
    a[0] += v.x; a[1] += v.y; a[2] += v.z; a[3] += v.w;
    b[0] += w.x; b[1] += w.y; b[2] += w.z; b[3] += w.w;
  }
}

template <int kBN>
__device__ __forceinline__ void reduce_rows_slice(const Params& p, int64_t m0, int n0, int r0, int r1, int tid,
                                                  double4* s_red /* kEpiWarps * 32 entries */) {
  constexpr int kC4 = kBN / 4;
  constexpr int kT = kEpiWarps * 32;
  const int items = (r1 - r0) * kC4;
  int G = 1;  // split groups: a power of two with G * items <= kT / 2, at least 4 splits per group
  while (G < 8 && 2 * G * items <= kT && 4 * G <= p.splits) G <<= 1;
  const double sc = p.out_scale;
  if (G == 1) {
    int idx = tid;
    for (; idx + kT < items; idx += 2 * kT) {  // items idx and idx + kT together
      const int64_t ra = m0 + r0 + idx / kC4, rb = m0 + r0 + (idx + kT) / kC4;
      const int ca = n0 + (idx % kC4) * 4, cb = n0 + ((idx + kT) % kC4) * 4;
      double a[4] = {0.0, 0.0, 0.0, 0.0}, b[4] = {0.0, 0.0, 0.0, 0.0};
      sum_splits2(p, p.c + ra * p.ldc + ca, p.c + rb * p.ldc + cb, 0, p.splits, a, b);
      *reinterpret_cast<float4*>(p.wout + ra * p.ldo + ca) =
          make_float4((float)(a[0] * sc), (float)(a[1] * sc), (float)(a[2] * sc), (float)(a[3] * sc));
      *reinterpret_cast<float4*>(p.wout + rb * p.ldo + cb) =
          make_float4((float)(b[0] * sc), (float)(b[1] * sc), (float)(b[2] * sc), (float)(b[3] * sc));
    }
    if (idx < items) {
      const int64_t r = m0 + r0 + idx / kC4;
      const int c = n0 + (idx % kC4) * 4;
      double a[4] = {0.0, 0.0, 0.0, 0.0};
      sum_splits<kBN>(p, p.c + r * p.ldc + c, 0, p.splits, a);
      *reinterpret_cast<float4*>(p.wout + r * p.ldo + c) =
          make_float4((float)(a[0] * sc), (float)(a[1] * sc), (float)(a[2] * sc), (float)(a[3] * sc));
    }
    return;
  }
  // one pass: thread (group gi, item idx); every epilogue thread reaches both barriers
  const int per = kT / G, gi = tid / per, idx = tid % per;
  const bool valid = idx < items;
  const int64_t r = m0 + r0 + idx / kC4;
  const int c = n0 + (idx % kC4) * 4;
  double a[4] = {0.0, 0.0, 0.0, 0.0};
  if (valid)
    sum_splits<kBN>(p, p.c + r * p.ldc + c, (int)((int64_t)gi * p.splits / G), (int)((int64_t)(gi + 1) * p.splits / G), a);
  s_red[tid] = make_double4(a[0], a[1], a[2], a[3]);
  epi_sync();
  if (gi == 0 && valid) {
    for (int g = 1; g < G; ++g) {  // group order
      const double4 t = s_red[g * per + idx];
      a[0] += t.x; a[1] += t.y; a[2] += t.z; a[3] += t.w;
    }
    *reinterpret_cast<float4*>(p.wout + r * p.ldo + c) =
        make_float4((float)(a[0] * sc), (float)(a[1] * sc), (float)(a[2] * sc), (float)(a[3] * sc));
  }
  epi_sync();
}

// Fused readout: a warp holds 32 consecutive rows (one per lane) x 32 columns.  A
// segmented inclusive scan over the lanes (segments = graphs, node rows of a graph are
// contiguous) leaves each graph's block sum on its last lane, which stores it: to
// pool_graph[g] when g lies wholly inside this 32-row block, else to the block's
// boundary slot (0: segment holding the block's first row, 1: the one holding its last).
// dippm_pool_combine adds the boundary slots of the blocks a graph spans, in block order.
// The warp's graph layout is the same for every column chunk of a tile: looked up once.
struct PoolRows {
  int gid;        // graph of this lane's row (-1 past M)
  bool uniform;   // all 32 rows in one graph
  float* whole;   // uniform case: pool_graph row of that graph if it lies inside the block, else
                  // the block's slot-0 partial row (column offset added per chunk)
};
__device__ __forceinline__ PoolRows pool_rows(const Params& p, int64_t row, int64_t r0) {
  PoolRows pr;
  pr.gid = row < p.M ? __ldg(p.node_graph + row) : -1;
  const int g0 = __shfl_sync(0xffffffffu, pr.gid, 0);
  pr.uniform = g0 >= 0 && __all_sync(0xffffffffu, pr.gid == g0);
  pr.whole = nullptr;
  if (pr.uniform) {
    const int gs = __ldg(p.graph_ptr + g0), ge = __ldg(p.graph_ptr + g0 + 1);
    pr.whole = ((gs >> 5) == ((ge - 1) >> 5)) ? p.pool_graph + (int64_t)g0 * p.N
                                               : p.pool_part + ((r0 >> 5) * 2 + 0) * p.N;  // gs <= r0 here
  }
  return pr;
}

__device__ __forceinline__ void pool_chunk(const Params& p, const PoolRows& pr, const float (&v)[32], int64_t r0,
                                           int n, int lane) {
  const int gid = pr.gid;
  if (pr.uniform) {
    // common case, all 32 rows in one graph: transpose-reduce (31 shuffles), lane L ends
    // with the block sum of column n + L, and the warp stores 128 contiguous bytes
    float t[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) t[i] = v[i];
#pragma unroll
    for (int k = 16; k >= 1; k >>= 1) {
      const bool upper = lane & k;
#pragma unroll
      for (int i = 0; i < k; ++i) {
        const float send = upper ? t[i] : t[i + k];
        const float recv = __shfl_xor_sync(0xffffffffu, send, k);
        t[i] = (upper ? t[i + k] : t[i]) + recv;
      }
    }
    pr.whole[n + lane] = t[0];
    return;
  }
  float s[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) s[i] = gid >= 0 ? v[i] : 0.f;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int gu = __shfl_up_sync(0xffffffffu, gid, off);
    const bool take = lane >= off && gu == gid;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float t = __shfl_up_sync(0xffffffffu, s[i], off);
      if (take) s[i] += t;
    }
  }
  const int gn = __shfl_down_sync(0xffffffffu, gid, 1);
  if (gid < 0 || (lane < 31 && gn == gid)) return;  // not the last row of its segment
  const int gs = __ldg(p.graph_ptr + gid), ge = __ldg(p.graph_ptr + gid + 1);
  float* dst;
  if ((gs >> 5) == ((ge - 1) >> 5)) {
    dst = p.pool_graph + (int64_t)gid * p.N + n;  // whole graph inside this block
  } else {
    const int64_t b = r0 >> 5;
    dst = p.pool_part + (b * 2 + (gs <= r0 ? 0 : 1)) * p.N + n;
  }
#pragma unroll
  for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4*>(dst + i) = make_float4(s[i], s[i + 1], s[i + 2], s[i + 3]);
}

// One persistent kernel for both tile shapes.  kCta == 2: a cluster of two
// CTAs on one TPC computes a 256 x kBN tile with cta_group::2 MMAs issued by the
// even CTA; each CTA stages its own 128 A rows and half of the kBN B rows, so
// per-SM operand traffic from L2 drops by a third against the 1-CTA 128 x kBN
// tile (the 1-CTA kernel is L2-bandwidth-bound; profiles/README.md).
template <int kFmt, bool kAMN, bool kBMN, int kBN, int kEpi, int kCta>
__global__ void __launch_bounds__(kThreads, 1)
    k_tc_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmC, Params p) {
  using C = Cfg<kFmt, kBN, kCta>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_stage = smem + C::kStages * C::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_stage + C::kEpiStage + C::kBiasBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = kCta == 2 ? cluster_rank() : 0u;
  const int cid = blockIdx.x / kCta, ncl = gridDim.x / kCta;
  if (p.ts && threadIdx.x == 0) p.ts[blockIdx.x * 8 + 0] = globaltimer();
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kEpiWarps * kCta);  // one arrival per epilogue warp of each CTA
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    if constexpr (kCta == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                   "r"(C::kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                   "r"(C::kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if constexpr (kCta == 2) cluster_sync_all();  // peer barriers initialised before any remote signal
  else __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  pdl_begin();  // barriers, TMEM and tensor maps are set up: now wait for the producer kernel
  if (p.ts && threadIdx.x == 0) p.ts[blockIdx.x * 8 + 1] = globaltimer();

  const int tiles_mn = p.m_tiles * p.n_tiles;
  const int total = tiles_mn * p.splits;
  const int kb_total = (int)((p.K + C::kBK - 1) / C::kBK);

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer (both CTAs; completion signalled on the leader's barrier) =====
      const uint32_t full_leader0 = kCta == 2 ? mapa(smem_u32(&full[0]), 0) : smem_u32(&full[0]);
      uint32_t it = 0;
      for (int t = cid; t < total; t += ncl) {
        const int split = t / tiles_mn, r = t % tiles_mn;
        const int m0 = (r / p.n_tiles) * C::kTileM + (int)rank * kBM;
        const int n0 = (r % p.n_tiles) * kBN + (int)rank * C::kBNl;
        const int kb0 = (int)((int64_t)split * kb_total / p.splits);
        const int kb1 = (int)((int64_t)(split + 1) * kb_total / p.splits);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % C::kStages;
          mbar_wait(&empty[s], ((it / C::kStages) & 1) ^ 1);
          uint8_t* sa = smem + s * C::kStageBytes;
          uint8_t* sb = sa + C::kPlanes * C::kATile;
          if (rank == 0) mbar_expect_tx(&full[s], C::kStageBytes * kCta);
          const uint32_t fb = full_leader0 + s * 8;
          const int k0 = kb * C::kBK;
#pragma unroll
          for (int pl = 0; pl < C::kPlanes; ++pl) {
            auto load = [&](void* dst, const CUtensorMap* map, int x, int y) {
              if constexpr (kCta == 2) tma_load_3d_pair(dst, map, fb, x, y, pl);
              else tma_load_3d(dst, map, &full[s], x, y, pl);
            };
            if constexpr (!kAMN) {
              load(sa + pl * C::kATile, &tmA, k0, m0);
            } else {
#pragma unroll
              for (int c = 0; c < kBM / C::kBK; ++c) load(sa + pl * C::kATile + c * C::kBK * 128, &tmA, m0 + c * C::kBK, k0);
            }
            if constexpr (!kBMN) {
              load(sb + pl * C::kBTile, &tmB, k0, n0);
            } else {
#pragma unroll
              for (int c = 0; c < C::kBNl / C::kBK; ++c)
                load(sb + pl * C::kBTile + c * C::kBK * 128, &tmB, n0 + c * C::kBK, k0);
            }
          }
        }
      }
      // tail: every MMA commit aimed at this CTA's empty barriers has landed before exit
      for (int i = 0; i < C::kStages; ++i, ++it) mbar_wait(&empty[it % C::kStages], ((it / C::kStages) & 1) ^ 1);
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ===== MMA issuer (one thread of the leader CTA) =====
      constexpr uint32_t idesc = make_idesc(kFmt, kAMN, kBMN, C::kTileM, kBN);
      constexpr uint32_t a_lbo = kAMN ? C::kBK * 128 : 16, b_lbo = kBMN ? C::kBK * 128 : 16;
      constexpr uint32_t a_step = kAMN ? C::kUK * 128 : 32, b_step = kBMN ? C::kUK * 128 : 32;
      // 32-bit MN-major operands use the 128B swizzle with 32-byte atoms
      // (UMMA layout 1 = SWIZZLE_128B_BASE32B, 4-row atoms of 512 B); all
      // others the plain 128B swizzle (layout 2, 8-row atoms of 1024 B).
      constexpr bool a32 = kAMN && kFmt == 2, b32 = kBMN && kFmt == 2;
      constexpr uint64_t a_lay = a32 ? 1 : 2, b_lay = b32 ? 1 : 2;
      constexpr uint32_t a_sbo = a32 ? 512 : 1024, b_sbo = b32 ? 512 : 1024;
      auto mma = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
        if constexpr (kCta == 2) umma_pair<kFmt>(d, a, b, idesc, acc);
        else umma<kFmt>(d, a, b, idesc, acc);
      };
      auto commit = [&](uint64_t* bar) {
        if constexpr (kCta == 2) umma_commit_pair(bar);
        else umma_commit(bar);
      };
      uint32_t it = 0, local = 0;
      for (int t = cid; t < total; t += ncl, ++local) {
        const int split = t / tiles_mn;
        const int kb0 = (int)((int64_t)split * kb_total / p.splits);
        const int kb1 = (int)((int64_t)(split + 1) * kb_total / p.splits);
        const uint32_t acc = local & 1, use = local >> 1;
        mbar_wait(&tempty[acc], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tbase + acc * kBN;
        uint32_t first = 1;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % C::kStages;
          mbar_wait(&full[s], (it / C::kStages) & 1);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * C::kStageBytes);
          const uint32_t sb = sa + C::kPlanes * C::kATile;
#pragma unroll
          for (int j = 0; j < C::kBK / C::kUK; ++j) {
            const uint64_t a_hi = sdesc(sa + j * a_step, a_lbo, a_sbo, a_lay);
            const uint64_t b_hi = sdesc(sb + j * b_step, b_lbo, b_sbo, b_lay);
            mma(d, a_hi, b_hi, first ? 0u : 1u);
            first = 0;
            if constexpr (C::kPlanes == 2) {
              const uint64_t a_lo = sdesc(sa + C::kATile + j * a_step, a_lbo, a_sbo, a_lay);
              const uint64_t b_lo = sdesc(sb + C::kBTile + j * b_step, b_lbo, b_sbo, b_lay);
              mma(d, a_hi, b_lo, 1u);
              mma(d, a_lo, b_hi, 1u);
            }
          }
          commit(&empty[s]);  // frees the smem slot (in both CTAs) when these MMAs retire
        }
        commit(&tfull[acc]);  // accumulator ready for the epilogue(s)
      }
    }
  } else {
    // ===== epilogue warps 2..9: TMEM lane quarter = warp % 4 =====
    const int q = warp & 3;            // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;  // two warps per quarter split the column chunks
    const uint32_t tempty_leader0 = kCta == 2 ? mapa(smem_u32(&tempty[0]), 0) : smem_u32(&tempty[0]);
    auto release = [&](uint32_t acc) {  // this warp is done reading accumulator `acc`
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (kCta == 2) mbar_arrive_cluster(tempty_leader0 + acc * 8);
        else mbar_arrive(&tempty[acc]);
      }
    };
    // the whole bias vector in shared memory once (packed FWD epilogue: 8 broadcast LDS.128 per chunk)
    const uint32_t s_bias = smem_u32(epi_stage + C::kEpiStage);
    if constexpr (C::kBiasCols > 0 && kEpi == EPI_FWD) {
      if (p.bias && p.N <= C::kBiasCols) {
        for (int c = threadIdx.x - 64; c < p.N; c += kEpiWarps * 32)
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(s_bias + 4 * c), "f"(__ldg(p.bias + c)) : "memory");
        epi_sync();
      }
    }
    uint32_t local = 0;
    for (int t = cid; t < total; t += ncl, ++local) {
      const int split = t / tiles_mn, r = t % tiles_mn;
      const int m0 = (r / p.n_tiles) * C::kTileM + (int)rank * kBM, n0 = (r % p.n_tiles) * kBN;
      const uint32_t acc = local & 1, use = local >> 1;
      const int64_t row = (int64_t)m0 + q * 32 + lane;
      if constexpr (kEpi == EPI_GATE) {
        if (p.gate_bits) {
          // 1-bit ReLU' masks written by the forward epilogue: one word per 32 columns.
          uint32_t gw[kBN / 64];
#pragma unroll
          for (int i = 0; i < kBN / 64; ++i)
            gw[i] = row < p.M ? __ldg(p.gate_bits + ((n0 >> 5) + half + 2 * i) * p.bits_ld + row) : 0u;
          mbar_wait(&tfull[acc], use & 1);
          tc_fence_after();
          const uint32_t tq = tbase + ((uint32_t)(q * 32) << 16) + acc * kBN;
          uint32_t rawb[2][32];
          tmem_ld32_issue(tq + half * 32, rawb[0]);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < kBN / 64; ++i) {
            const int ch = half + 2 * i;
            if (i + 1 < kBN / 64) tmem_ld32_issue(tq + (ch + 2) * 32, rawb[(i + 1) & 1]);
            uint32_t(&raw)[32] = rawb[i & 1];
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = (gw[i] >> j) & 1u ? __uint_as_float(raw[j]) * p.gate_scale : 0.f;
            epi_store_chunk(epi_stage + (warp - 2) * kStageWarpBytes, &tmC, p.out.dtype, lane, v, n0 + ch * 32,
                            m0 + q * 32, local * (kBN / 64) + i);
            tmem_wait_ld();
          }
          release(acc);
          continue;
        }
        // The gate (activation of the layer below) is streamed one 32-column
        // chunk ahead: chunk 0 is fetched while the MMAs are still running.
        uint4 graw[8];
        if (row < p.M) gate_issue<kFmt>(p.gate, row, n0 + half * 32, graw);
        mbar_wait(&tfull[acc], use & 1);
        tc_fence_after();
        uint32_t gm = row < p.M ? gate_mask<kFmt>(p.gate, row, n0 + half * 32, graw) : 0u;
#pragma unroll 1
        for (int ch = half; ch < kBN / 32; ch += 2) {
          const bool more = ch + 2 < kBN / 32 && row < p.M;
          if (more) gate_issue<kFmt>(p.gate, row, n0 + (ch + 2) * 32, graw);
          uint32_t raw[32];
          tmem_ld32(tbase + ((uint32_t)(q * 32) << 16) + acc * kBN + ch * 32, raw);
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = (gm >> i) & 1u ? __uint_as_float(raw[i]) * p.gate_scale : 0.f;
          epi_store_chunk(epi_stage + (warp - 2) * kStageWarpBytes, &tmC, p.out.dtype, lane, v, n0 + ch * 32,
                          m0 + q * 32, local * (kBN / 64) + (ch >> 1));
          if (more) gm = gate_mask<kFmt>(p.gate, row, n0 + (ch + 2) * 32, graw);
        }
        release(acc);
        continue;
      }
      // fused readout: this warp's graph layout, looked up before the accumulator is ready
      PoolRows pr{};
      if constexpr (kEpi == EPI_FWD)
        if (p.pool_part) pr = pool_rows(p, row, m0 + q * 32);
      // 1-CTA tiles (short-K layer 1: the epilogue is the bottleneck): lane l holds bias column l
      // of each of this warp's chunks, fetched before the accumulator wait and broadcast with
      // shuffles, so no load latency sits inside the chunk loop.  Pair tiles (long K, epilogue
      // hidden under the MMAs) load the bias per chunk: fewer instructions.
      // packed FWD epilogue: bf16 output with bias and ReLU and no fused readout (layers 1-2)
      // (1-CTA tiles only: compiled into the pair kernel, the packed path made its register
      // allocation spill, which cost the layer-3 readout epilogue more than layer 2 gained)
      const bool fast_fwd = kFmt == 1 && kEpi == EPI_FWD && kCta == 1 && p.out.base && p.out.dtype == DIPPM_DT_BF16 &&
                            p.relu && p.bias && !p.pool_part && (C::kBiasCols == 0 || p.N <= C::kBiasCols) &&
                            !(p.dbg & 8);
      float bl[kBN / 64];
      if constexpr ((kEpi == EPI_FWD || kEpi == EPI_FWD_DROP) && kCta == 1) {
        if (!fast_fwd) {
#pragma unroll
          for (int i = 0; i < kBN / 64; ++i) bl[i] = p.bias ? __ldg(p.bias + n0 + (half + 2 * i) * 32 + lane) : 0.f;
        }
      }
      mbar_wait(&tfull[acc], use & 1);
      tc_fence_after();
      if (p.ts && threadIdx.x == 64 && local == 0) p.ts[blockIdx.x * 8 + 4] = globaltimer();
      if (p.dbg & 4) {
        release(acc);
        continue;
      }
      // TMEM reads run one chunk ahead: chunk i+1 is in flight while chunk i is processed.
      const uint32_t tq = tbase + ((uint32_t)(q * 32) << 16) + acc * kBN;
      uint32_t rawb[2][32];
      tmem_ld32_issue(tq + half * 32, rawb[0]);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < kBN / 64; ++i) {
        const int ch = half + 2 * i;
        if (i + 1 < kBN / 64) tmem_ld32_issue(tq + (ch + 2) * 32, rawb[(i + 1) & 1]);
        uint32_t(&raw)[32] = rawb[i & 1];
        const int n = n0 + ch * 32;
        if (kEpi == EPI_FWD && fast_fwd) {
          // bf16 output + bias + ReLU, no readout: the packed sequence (see pos_bits_bf16x2)
          uint32_t w[16];
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            const float4 b = C::kBiasCols ? lds128f(s_bias + (uint32_t)(n * 4 + g * 16))  // broadcast
                                          : __ldg(reinterpret_cast<const float4*>(p.bias + n) + g);
            const float2 x0 = add_f32x2(make_float2(__uint_as_float(raw[4 * g]), __uint_as_float(raw[4 * g + 1])),
                                        make_float2(b.x, b.y));
            const float2 x1 = add_f32x2(make_float2(__uint_as_float(raw[4 * g + 2]), __uint_as_float(raw[4 * g + 3])),
                                        make_float2(b.z, b.w));
            w[2 * g] = relu_bf16x2(pack_bf16x2(x0.x, x0.y));
            w[2 * g + 1] = relu_bf16x2(pack_bf16x2(x1.x, x1.y));
          }
          if (p.relu_bits && row < p.M && !(p.dbg & 2)) {
            const uint32_t bits = pos_bits32(w);
            if (p.bits_ld > 0) p.relu_bits[(n >> 5) * p.bits_ld + row] = bits;
            else p.relu_bits[row * (p.N >> 5) + (n >> 5)] = bits;
          }
          if (!(p.dbg & 1))
            epi_store_packed(epi_stage + (warp - 2) * kStageWarpBytes, &tmC, lane, w, n, m0 + q * 32,
                             local * (kBN / 64) + (ch >> 1));
          else if (w[0] == 0x12345678u && w[15] == 0x9abcdef0u)  // keep the values live
            p.relu_bits[0] = w[3];
        } else if constexpr (kEpi == EPI_FWD || kEpi == EPI_FWD_DROP) {
          float v[32];
          if constexpr (kCta == 1) {
#pragma unroll
            for (int k = 0; k < 32; ++k) v[k] = __shfl_sync(0xffffffffu, bl[i], k);
          } else if (p.bias) {
#pragma unroll
            for (int g = 0; g < 8; ++g) {
              const float4 b4 = __ldg(reinterpret_cast<const float4*>(p.bias + n) + g);
              v[4 * g] = b4.x; v[4 * g + 1] = b4.y; v[4 * g + 2] = b4.z; v[4 * g + 3] = b4.w;
            }
          } else {
#pragma unroll
            for (int k = 0; k < 32; ++k) v[k] = 0.f;
          }
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const float x = __uint_as_float(raw[k]) + v[k];
            v[k] = p.relu ? fmaxf(x, 0.f) : x;
          }
          if constexpr (kEpi == EPI_FWD_DROP) {  // inverted dropout after ReLU (gnn.py:277-281)
            const uint64_t seed = p.seed ^ (p.seed_dev ? (uint64_t)p.seed_dev[0] * 0x9E3779B97F4A7C15ull : 0ull);
            if (row < p.M) {
              if (p.drop_mode == 1) {
#pragma unroll
                for (int i = 0; i < 32; i += 4) {
                  const float4 m4 = *reinterpret_cast<const float4*>(p.mask + row * p.ldm + n + i);
                  v[i] *= m4.x; v[i + 1] *= m4.y; v[i + 2] *= m4.z; v[i + 3] *= m4.w;
                }
              } else {  // counter-hash stream (numerics.py:45-55 semantics, statistical parity)
                const float keep = 1.0f / (1.0f - p.drop_p);
#pragma unroll 8
                for (int i = 0; i < 32; ++i) {
                  const int64_t idx = row * p.ldm + n + i;
                  const float mk = uniform_hash(seed, (uint64_t)idx) >= p.drop_p ? keep : 0.f;
                  v[i] *= mk;
                }
                if (p.mask) {  // optional record of the mask (the backward uses the 1-bit masks)
#pragma unroll
                  for (int i = 0; i < 32; i += 4) {
                    float4 m4;
                    m4.y = uniform_hash(seed, (uint64_t)(row * p.ldm + n + i + 1)) >= p.drop_p ? keep : 0.f;
                    m4.z = uniform_hash(seed, (uint64_t)(row * p.ldm + n + i + 2)) >= p.drop_p ? keep : 0.f;
                    m4.w = uniform_hash(seed, (uint64_t)(row * p.ldm + n + i + 3)) >= p.drop_p ? keep : 0.f;
                    m4.x = uniform_hash(seed, (uint64_t)(row * p.ldm + n + i)) >= p.drop_p ? keep : 0.f;
                    *reinterpret_cast<float4*>(p.mask + row * p.ldm + n + i) = m4;
                  }
                }
              }
            }
          }
          if (p.relu_bits && row < p.M) {  // 1-bit ReLU' (and dropout) mask for the backward GATE epilogue
            uint32_t bits = 0;
#pragma unroll
            for (int i = 0; i < 32; ++i) bits |= (uint32_t)(v[i] > 0.f) << i;
            if (p.bits_ld > 0) p.relu_bits[(n >> 5) * p.bits_ld + row] = bits;  // chunk-major: 128 B per warp
            else p.relu_bits[row * (p.N >> 5) + (n >> 5)] = bits;  // row-major (bits_ld 0): read per row
          }
          if (p.pool_part) pool_chunk(p, pr, v, m0 + q * 32, n, lane);  // fused readout (K4, gnn.py:214)
          if (p.out.base)
            epi_store_chunk(epi_stage + (warp - 2) * kStageWarpBytes, &tmC, p.out.dtype, lane, v, n, m0 + q * 32,
                            local * (kBN / 64) + (ch >> 1));
        } else {
          // fp32 rows (weight-gradient split partials or final output, STORE): staged through this
          // warp's 4 KB slot (128B-swizzled 16-byte units) and written 4 rows per instruction,
          // 8 lanes x 16 B per row -- coalesced 128-byte row pieces instead of a 16-byte piece of
          // each of 32 rows per instruction (the partial rows were LSU-transaction bound)
          const bool fin = kEpi == EPI_PARTIAL && p.reduce_mode == 3;  // single split: final output, scaled
          float4* st = reinterpret_cast<float4*>(epi_stage + (warp - 2) * kStageWarpBytes);
          __syncwarp();  // the previous chunk's reads of the slot are done
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            float4 f = make_float4(__uint_as_float(raw[4 * g]), __uint_as_float(raw[4 * g + 1]),
                                   __uint_as_float(raw[4 * g + 2]), __uint_as_float(raw[4 * g + 3]));
            if (fin)
              f = make_float4((float)(f.x * p.out_scale), (float)(f.y * p.out_scale), (float)(f.z * p.out_scale),
                              (float)(f.w * p.out_scale));
            st[lane * 8 + (g ^ (lane & 7))] = f;
          }
          __syncwarp();
          float* base = fin ? p.wout : p.c + (kEpi == EPI_PARTIAL ? (int64_t)split * p.M * p.ldc : 0);
          const int64_t ld = fin ? p.ldo : p.ldc;
          const int u = lane & 7;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int rr = (lane >> 3) + 4 * k;
            const int64_t grow = m0 + q * 32 + rr;
            const float4 val = st[rr * 8 + (u ^ (rr & 7))];
            if (grow < p.M) *reinterpret_cast<float4*>(base + grow * ld + n + 4 * u) = val;
          }
        }
        tmem_wait_ld();  // chunk i+1 has landed
      }
      release(acc);
      if constexpr (kEpi == EPI_PARTIAL) {
        if (p.reduce_mode == 1 || p.reduce_mode == 2) {
          // ---- fused split-K reduction (replaces a separate reduce kernel) ----
          const int tid = threadIdx.x - 64;
          int* arrive = p.sync + r * kCta + rank;
          int* depart = arrive + tiles_mn * kCta;
          __shared__ uint32_t s_go;  // "this CTA reduces" flag, away from the TMEM address slot
          uint32_t* s_flag = &s_go;
          epi_sync();  // this CTA's partial rows are all written
          if (p.ts && tid == 0) p.ts[blockIdx.x * 8 + 5] = globaltimer();
          if (tid == 0) {
            __threadfence();
            const int old = atomicAdd(arrive, 1);
            uint32_t go = 1;
            if (p.reduce_mode == 1) {
              uint32_t spins = 0;
              uint64_t t0 = 0;
              while (ld_acquire(arrive) < p.splits) {
                if (++spins == 64) t0 = globaltimer();
                if (spins > 64 && (spins & 255) == 0 && globaltimer() - t0 > 2000000000ull) __trap();
              }
            } else {
              go = old == p.splits - 1;
              if (go) __threadfence();
            }
            *s_flag = go;
          }
          epi_sync();
          if (p.ts && tid == 0) p.ts[blockIdx.x * 8 + 6] = globaltimer();
          const int rows_valid = (int)(p.M - m0 < kBM ? p.M - m0 : kBM);
          if (*s_flag && rows_valid > 0) {
            const int r0 = p.reduce_mode == 1 ? (int)((int64_t)split * rows_valid / p.splits) : 0;
            const int r1 = p.reduce_mode == 1 ? (int)((int64_t)(split + 1) * rows_valid / p.splits) : rows_valid;
            reduce_rows_slice<kBN>(p, m0, n0, r0, r1, tid, reinterpret_cast<double4*>(epi_stage));
          }
          if (p.reduce_mode == 1) {
            epi_sync();
            if (tid == 0 && atomicAdd(depart, 1) == p.splits - 1) {  // every split is past its spin
              *arrive = 0;
              *depart = 0;
            }
          } else if (tid == 0 && *s_flag) {
            *arrive = 0;  // the last arriver: all splits have arrived
          }
        }
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // TMA stores drained
    if constexpr (kEpi == EPI_PARTIAL) {
      // deferred bias fold (gnn.py:230): the layer's agg^T kernel left per-block column sums of dz;
      // CTA b folds float4 column group b (b, b + grid, ...): every thread sums its rows in row
      // order, the 256 thread sums meet in shared memory in thread order -- deterministic
      if (p.bias_part) {
        const int tid = threadIdx.x - 64;
        const int rows = __ldcg(p.bias_count);
        double4* s_red = reinterpret_cast<double4*>(epi_stage);  // staging is idle now (stores drained)
        for (int g4 = blockIdx.x; g4 < (int)(p.N / 4); g4 += gridDim.x) {
          double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
          for (int r = tid; r < rows; r += kEpiWarps * 32) {
            const float4 v = __ldcg(reinterpret_cast<const float4*>(p.bias_part + (int64_t)r * p.N) + g4);
            a0 += v.x; a1 += v.y; a2 += v.z; a3 += v.w;
          }
#pragma unroll
          for (int o = 16; o; o >>= 1) {  // fixed xor tree within the warp, then the warps in order
            a0 += __shfl_xor_sync(0xffffffffu, a0, o);
            a1 += __shfl_xor_sync(0xffffffffu, a1, o);
            a2 += __shfl_xor_sync(0xffffffffu, a2, o);
            a3 += __shfl_xor_sync(0xffffffffu, a3, o);
          }
          epi_sync();
          if (lane == 0) s_red[tid >> 5] = make_double4(a0, a1, a2, a3);
          epi_sync();
          if (tid < 4) {
            double t = 0.0;
            for (int w = 0; w < kEpiWarps; ++w) {
              const double4 q = s_red[w];
              t += tid == 0 ? q.x : (tid == 1 ? q.y : (tid == 2 ? q.z : q.w));
            }
            p.bias_fold[g4 * 4 + tid] = (float)t;
          }
        }
      }
    }
  }
  if (p.ts && threadIdx.x == 64) p.ts[blockIdx.x * 8 + 2] = globaltimer();  // first epilogue thread done
  tc_fence_before();
  if constexpr (kCta == 2) cluster_sync_all();  // both CTAs done with TMEM and with remote barriers
  else __syncthreads();
  if (p.ts && threadIdx.x == 0) p.ts[blockIdx.x * 8 + 3] = globaltimer();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (kCta == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(C::kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(C::kTmemCols));
  }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

// 3-D map over (cols, rows, plane) of a row-major operand; box = one 128-byte
// swizzle row of columns by box_rows rows.
static int make_map(CUtensorMap* map, const dippm_act_t& v, int64_t rows, int64_t cols, int box_cols, int box_rows,
                    bool atom32 = false, bool store_map = false) {
  auto fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return DIPPM_ERR_CUDA;
  }
  const int elem = v.dtype == DIPPM_DT_BF16 ? 2 : 4;
  const int planes = v.dtype == DIPPM_DT_TF32X3 ? 2 : 1;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)planes};
  int64_t pstride = planes == 2 ? v.plane_stride : rows * v.ld;
  cuuint64_t strides[2] = {(cuuint64_t)(v.ld * elem), (cuuint64_t)(pstride * elem)};
  cuuint32_t box[3] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, v.dtype == DIPPM_DT_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                  3, v.data, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  // epilogue store maps: 32-column boxes, 64 B rows (bf16) -> 64B swizzle, 128 B rows -> 128B
                  store_map ? (elem == 2 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B)
                            : (atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B),
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): rows=%lld cols=%lld ld=%lld box=%dx%d", (int)r, (long long)rows,
              (long long)cols, (long long)v.ld, box_cols, box_rows);
    return DIPPM_ERR_ARG;
  }
  return DIPPM_OK;
}

template <int kFmt, bool kAMN, bool kBMN, int kBN, int kEpi, int kCta>
static int run(const dippm_gemm_args_t* a, cudaStream_t s) {
  using Cf = Cfg<kFmt, kBN, kCta>;
  auto kern = k_tc_gemm<kFmt, kAMN, kBMN, kBN, kEpi, kCta>;
  static bool attr_set = false;
  if (!attr_set) {
    DIPPM_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::kSmemBytes));
    attr_set = true;
  }
  CUtensorMap ma, mb, mc;
  int st;
  // A logical (M x K); B logical (N x K).  Boxes are per CTA (B: kBN / kCta rows).
  if (!kAMN) st = make_map(&ma, a->a, a->M, a->K, Cf::kBK, kBM);
  else st = make_map(&ma, a->a, a->K, a->M, Cf::kBK, Cf::kBK, kFmt == 2);
  if (st) return st;
  if (!kBMN) st = make_map(&mb, a->b, a->N, a->K, Cf::kBK, Cf::kBNl);
  else st = make_map(&mb, a->b, a->K, a->N, Cf::kBK, Cf::kBK, kFmt == 2);
  if (st) return st;
  Params p{};
  p.M = a->M;
  p.N = a->N;
  p.K = a->K;
  const int kb_total = ceil_div_i(a->K, Cf::kBK);
  p.splits = kEpi == EPI_PARTIAL ? (int)std::max<int64_t>(1, a->splits) : 1;
  if (p.splits > kb_total) {
    set_error("gemm: %d splits exceed %d k-blocks (use dippm_wgrad_splits)", p.splits, kb_total);
    return DIPPM_ERR_ARG;
  }
  p.m_tiles = ceil_div_i(a->M, Cf::kTileM);
  p.n_tiles = (int)(a->N / kBN);
  p.bias = a->bias;
  p.relu = (int)a->relu;
  p.out = make_view(a->out);
  p.c = a->c;
  p.ldc = a->ldc;
  p.gate = make_view(a->gate);
  p.gate_scale = (float)a->gate_scale;
  p.drop_mode = (int)a->drop_mode;
  p.mask = a->mask;
  p.ldm = a->ldm;
  p.drop_p = (float)a->drop_p;
  p.seed = a->seed;
  p.seed_dev = a->seed_dev;
  p.relu_bits = a->relu_bits;
  p.pool_part = a->pool_partial;
  p.pool_graph = a->pool_graph;
  p.node_graph = a->node_graph;
  p.graph_ptr = a->graph_ptr;
  p.gate_bits = a->gate_bits;
  p.bits_ld = a->bits_ld;
  if (kEpi == EPI_PARTIAL && a->bias_partial) {
    if (!a->bias_grad) {
      set_error("gemm WGRAD: bias_partial needs bias_grad");
      return DIPPM_ERR_ARG;
    }
    p.bias_part = a->bias_partial;
    p.bias_count = dippm_colsum_count_slot(const_cast<float*>(a->bias_partial), a->K, (int32_t)a->N);
    p.bias_fold = a->bias_grad;
  }
  static const int dbg = getenv("DIPPM_GEMM_DEBUG") ? atoi(getenv("DIPPM_GEMM_DEBUG")) : 0;
  p.dbg = dbg;
  static unsigned long long* ts = getenv("DIPPM_GEMM_TS") ? (unsigned long long*)strtoull(getenv("DIPPM_GEMM_TS"), nullptr, 0) : nullptr;
  p.ts = ts;
  const int total = p.m_tiles * p.n_tiles * p.splits;
  const int clusters = std::min(total, num_sms() / kCta);
  p.reduce_mode = 0;
  if (kEpi == EPI_PARTIAL && a->tile_sync) {
    if (a->out.dtype != DIPPM_DT_F32 || !a->out.data || (p.splits > 1 && !a->c)) {
      set_error("gemm WGRAD fused reduce: needs an F32 out view and (splits > 1) a partial workspace c");
      return DIPPM_ERR_ARG;
    }
    p.reduce_mode = p.splits == 1 ? 3 : (total <= clusters ? 1 : 2);
    p.wout = reinterpret_cast<float*>(a->out.data);
    p.ldo = a->out.ld;
    p.out_scale = a->out_scale;
    p.sync = a->tile_sync;
  }
  if ((kEpi == EPI_FWD || kEpi == EPI_FWD_DROP || kEpi == EPI_GATE) && a->out.data) {
    st = make_map(&mc, a->out, a->M, a->N, 32, 32, false, true);  // epilogue TMA-store target
    if (st) return st;
  } else {
    mc = ma;  // unused
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(clusters * kCta);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = Cf::kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (kCta == 2) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = kCta;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  DIPPM_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, ma, mb, mc, p));
  DIPPM_LAUNCH_CHECK("k_tc_gemm");
  return DIPPM_OK;
}

// ---------------------------------------------------------------------------------------
// Short-K forward (layer 1: z = [X | agg X] @ W1 + b, K = 64): the MMAs are trivial and the
// kernel is bound by its epilogue (bias + ReLU + bf16 rounding + 1-bit masks + 78 MB of stores),
// which the general kernel runs with only 8 epilogue warps (2 per scheduler: latency-bound at
// ~0.4 IPC).  Here one warp does TMA + MMA and 16 warps drain the accumulators (4 per TMEM lane
// quarter, 2 of a tile's 8 column chunks each); the whole B (W1, N x 64) stays resident in
// shared memory, A streams through a 6-deep ring of 128 x 64 k-blocks, and the two 256-column
// TMEM accumulators alternate between tiles.
namespace sk {
constexpr int kEpi = 16;                 // epilogue warps
constexpr int kThreads = 32 * (1 + kEpi);
constexpr int kBN = 256;                 // tile columns (one accumulator)
constexpr int kStages = 5;
constexpr int kATile = kBM * 128;        // 128 rows x 64 bf16
constexpr int kMaxN = 512;
constexpr int kBBytes = kMaxN * 128;     // N rows x 64 bf16 (MN-major boxes of 64 x 64)
constexpr int kStage = kEpi * 4096;
constexpr int kSmem = kBBytes + kStages * kATile + kStage + kMaxN * 4 + 1024 + 256;
}  // namespace sk

__global__ void __launch_bounds__(sk::kThreads, 1)
    k_fwd_shortk(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmC, Params p) {
  using namespace sk;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int nb = (int)p.N / 64;                 // 64-column boxes of B
  uint8_t* sB = smem;                           // [nb][64 k-rows x 128 B]
  uint8_t* sA = sB + nb * 8192;
  uint8_t* stage = sA + kStages * kATile;
  float* s_bias = reinterpret_cast<float*>(stage + kStage);
  uint64_t* full = reinterpret_cast<uint64_t*>(s_bias + p.N);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* bfull = tempty + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kEpi);
    }
    mbar_init(bfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  pdl_begin();
  if (warp > 0) {  // the bias (written by the previous step's Adam kernel) once, into shared memory
    for (int c = threadIdx.x - 32; c < p.N; c += kEpi * 32) s_bias[c] = __ldg(p.bias + c);
    asm volatile("bar.sync 1, %0;" ::"n"(kEpi * 32) : "memory");
  }
  const int n_tiles = (int)p.N / kBN;
  const int total = p.m_tiles * n_tiles;
  if (warp == 0) {
    if (lane == 0) {
      // B once: nb boxes of (64 N-columns x 64 K-rows), MN-major, 128B swizzle
      mbar_expect_tx(bfull, nb * 8192);
      for (int c = 0; c < nb; ++c) tma_load_3d(sB + c * 8192, &tmB, bfull, c * 64, 0, 0);
      constexpr uint32_t idesc = make_idesc(1, false, true, kBM, kBN);
      uint32_t it_load = 0, it_mma = 0, local = 0;
      // A k-blocks are fetched up to kStages tiles ahead of the MMAs (one k-block per tile)
      auto issue_load = [&](int t) {
        const int s = it_load % kStages;
        mbar_wait(&empty[s], ((it_load / kStages) & 1) ^ 1);
        mbar_expect_tx(&full[s], kATile);
        tma_load_3d(sA + s * kATile, &tmA, &full[s], 0, (t / n_tiles) * kBM, 0);
        ++it_load;
      };
      int t_load = blockIdx.x;
      for (int k = 0; k < kStages && t_load < total; ++k, t_load += gridDim.x) issue_load(t_load);
      mbar_wait(bfull, 0);
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
        const uint32_t acc = local & 1, use = local >> 1;
        const int n0 = (t % n_tiles) * kBN;
        const int s = it_mma % kStages;
        mbar_wait(&tempty[acc], (use & 1) ^ 1);
        mbar_wait(&full[s], (it_mma / kStages) & 1);
        tc_fence_after();
        const uint32_t a0 = smem_u32(sA + s * kATile), b0 = smem_u32(sB + (n0 / 64) * 8192);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          umma<1>(tbase + acc * kBN, sdesc(a0 + j * 32, 16, 1024), sdesc(b0 + j * 2048, 8192, 1024), idesc, j > 0);
        umma_commit(&empty[s]);
        umma_commit(&tfull[acc]);
        // refill the slot the PREVIOUS tile used (its MMAs have had a tile's time to retire), so
        // this thread never waits on the MMAs it has just issued
        if (it_mma > 0 && t_load < total) {
          issue_load(t_load);
          t_load += gridDim.x;
        }
        ++it_mma;
      }
      for (int i = 0; i < kStages; ++i, ++it_load) mbar_wait(&empty[it_load % kStages], ((it_load / kStages) & 1) ^ 1);
    }
  } else {
    const int e = warp - 1;
    const int q = warp & 3;          // TMEM lane quarter this warp may read
    const int sub = (warp - 1) >> 2;  // 0..3: chunks sub and sub + 4 of each tile
    uint8_t* stg = stage + e * 4096;
    const uint32_t sb = smem_u32(s_bias);
    uint32_t local = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
      const uint32_t acc = local & 1, use = local >> 1;
      const int m0 = (t / n_tiles) * kBM, n0 = (t % n_tiles) * kBN;
      const int64_t row = (int64_t)m0 + q * 32 + lane;
      mbar_wait(&tfull[acc], use & 1);
      tc_fence_after();
      const uint32_t tq = tbase + ((uint32_t)(q * 32) << 16) + acc * kBN;
      uint32_t raw[2][32];
      tmem_ld32_issue(tq + sub * 32, raw[0]);
      tmem_ld32_issue(tq + (sub + 4) * 32, raw[1]);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);  // the accumulator is in registers: the MMAs may go on
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int n = n0 + (sub + 4 * i) * 32;
        uint32_t w[16];
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          const float4 b = lds128f(sb + (uint32_t)(n * 4 + g * 16));
          const float2 x0 = add_f32x2(make_float2(__uint_as_float(raw[i][4 * g]), __uint_as_float(raw[i][4 * g + 1])),
                                      make_float2(b.x, b.y));
          const float2 x1 = add_f32x2(make_float2(__uint_as_float(raw[i][4 * g + 2]), __uint_as_float(raw[i][4 * g + 3])),
                                      make_float2(b.z, b.w));
          w[2 * g] = relu_bf16x2(pack_bf16x2(x0.x, x0.y));
          w[2 * g + 1] = relu_bf16x2(pack_bf16x2(x1.x, x1.y));
        }
        if (p.relu_bits && row < p.M) p.relu_bits[(n >> 5) * p.bits_ld + row] = pos_bits32(w);
        epi_store_packed(stg, &tmC, lane, w, n, m0 + q * 32, i);
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
  }
}

static bool shortk_ok(const dippm_gemm_args_t* a) {
  return a->kind == DIPPM_GEMM_FWD && a->a.dtype == DIPPM_DT_BF16 && a->K == 64 && a->b_mn_major && !a->drop_mode &&
         a->relu && a->bias && a->out.data && a->out.dtype == DIPPM_DT_BF16 && !a->pool_partial && a->N % sk::kBN == 0 &&
         a->N <= sk::kMaxN && (!a->relu_bits || a->bits_ld >= a->M) && a->cta_pair == 0 && !getenv("DIPPM_NO_SHORTK");
}

static int run_shortk(const dippm_gemm_args_t* a, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    DIPPM_CUDA_CHECK(cudaFuncSetAttribute(k_fwd_shortk, cudaFuncAttributeMaxDynamicSharedMemorySize, sk::kSmem));
    attr_set = true;
  }
  CUtensorMap ma, mb, mc;
  int st = make_map(&ma, a->a, a->M, a->K, 64, kBM);
  if (!st) st = make_map(&mb, a->b, a->K, a->N, 64, 64);
  if (!st) st = make_map(&mc, a->out, a->M, a->N, 32, 32, false, true);
  if (st) return st;
  Params p{};
  p.M = a->M;
  p.N = a->N;
  p.K = a->K;
  p.m_tiles = ceil_div_i(a->M, kBM);
  p.n_tiles = (int)(a->N / sk::kBN);
  p.bias = a->bias;
  p.relu = 1;
  p.out = make_view(a->out);
  p.relu_bits = a->relu_bits;
  p.bits_ld = a->bits_ld;
  const int total = p.m_tiles * p.n_tiles;
  DIPPM_LAUNCH_PDL(k_fwd_shortk, dim3(std::min(total, num_sms())), dim3(sk::kThreads), (size_t)sk::kSmem, s, ma, mb, mc, p);
  DIPPM_LAUNCH_CHECK("k_fwd_shortk");
  return DIPPM_OK;
}

// Tile choice: 256 x 256 CTA-pair tiles when M is large (the SAGE layers,
// M = nodes), 1-CTA 128 x BN tiles otherwise; narrower BN for short problems
// (the FC head, M = #graphs) so more CTAs run.
template <int kFmt, bool kAMN, bool kBMN, int kEpi>
static int run_bn(const dippm_gemm_args_t* a, cudaStream_t s) {
  const int64_t m_tiles = ceil_div_i(a->M, kBM);
  const bool pair_ok = a->N % 256 == 0;
  const int64_t splits = kEpi == EPI_PARTIAL ? std::max<int64_t>(1, a->splits) : 1;
  const bool pair = a->cta_pair == 2 ? pair_ok
                                     : (a->cta_pair != 1 && pair_ok && a->M > kBM &&
                                        (kEpi == EPI_PARTIAL || a->K > 128) &&  // short K: epilogue-bound, 1-CTA wins
                                        4 * m_tiles * (a->N / 256) * splits >= 3 * num_sms());
  if (a->cta_pair == 2 && !pair_ok) {
    set_error("gemm: cta_pair=2 needs N %% 256 == 0 (N=%lld)", (long long)a->N);
    return DIPPM_ERR_ARG;
  }
  if (pair) return run<kFmt, kAMN, kBMN, 256, kEpi, 2>(a, s);
  const bool narrow = (kEpi != EPI_PARTIAL || splits == 1) && m_tiles * (a->N / 256) < num_sms() / 2;
  if (a->N % 256 == 0 && !narrow) return run<kFmt, kAMN, kBMN, 256, kEpi, 1>(a, s);
  if (a->N % 128 == 0 && !(narrow && m_tiles * (a->N / 128) < num_sms() / 2))
    return run<kFmt, kAMN, kBMN, 128, kEpi, 1>(a, s);
  return run<kFmt, kAMN, kBMN, 64, kEpi, 1>(a, s);
}

template <int kFmt>
static int dispatch(const dippm_gemm_args_t* a, cudaStream_t s) {
  switch (a->kind) {
    case DIPPM_GEMM_FWD:
      if (a->drop_mode) return run_bn<kFmt, false, true, EPI_FWD_DROP>(a, s);  // head fc1/fc2 in train mode
      return a->b_mn_major ? run_bn<kFmt, false, true, EPI_FWD>(a, s) : run_bn<kFmt, false, false, EPI_FWD>(a, s);
    case DIPPM_GEMM_GATE: return run_bn<kFmt, false, false, EPI_GATE>(a, s);
    case DIPPM_GEMM_STORE: return run_bn<kFmt, false, false, EPI_STORE>(a, s);
    default: return run_bn<kFmt, true, true, EPI_PARTIAL>(a, s);
  }
}

// 128B-swizzled 3-D tensor map of a row-major operand (cols, rows, plane); box = box_cols x
// box_rows.  For kernels in other translation units (the tensor-core FC head).
int make_map_sw128(CUtensorMap* map, const dippm_act_t& v, int64_t rows, int64_t cols, int box_cols, int box_rows) {
  return make_map(map, v, rows, cols, box_cols, box_rows);
}

}  // namespace tc
}  // namespace dippm

using namespace dippm;

extern "C" int32_t dippm_gemm_simt_impl(const dippm_gemm_args_t* a, cudaStream_t s);

extern "C" int32_t dippm_wgrad_splits(int64_t M, int64_t N, int64_t K) {
  const int bn = N % 256 == 0 ? 256 : (N % 128 == 0 ? 128 : 64);
  const int64_t tiles = (int64_t)ceil_div_i(M, tc::kBM) * (N / bn);
  const int kb_total = ceil_div_i(K, 64);  // bf16 k-block; tf32 uses 32-row blocks (twice as many)
  // Short reductions (the head's K = #graphs): no split — narrow output tiles supply the
  // parallelism and the epilogue stores the result directly (no partials, no reduce).
  if (kb_total <= 8) return 1;
  int want = (int)std::max<int64_t>(1, num_sms() / std::max<int64_t>(1, tiles));
  // tiny outputs (layer 1: 65 x 512 = 2 tiles) stream almost nothing per split beyond their
  // partial tile, so the split-K partials and their reduction dominate: 64 splits measured
  // 26.9 us against 29.2 us for 74 (the GPU-filling count) at configs[1]
  if (tiles <= 2) want = std::min(want, 64);
  return std::min(want, kb_total);  // every split owns >= 1 k-block for both k-block sizes
}

extern "C" int64_t dippm_wgrad_sync_ints(int64_t M, int64_t N) {
  return 2 * (int64_t)ceil_div_i(M, tc::kBM) * ceil_div_i(N, 64);  // arrive + depart per (tile, CTA)
}

extern "C" int32_t dippm_gemm(const dippm_gemm_args_t* a, int32_t backend, void* stream) {
  DIPPM_ARG_CHECK(a != nullptr, "gemm: null args");
  DIPPM_ARG_CHECK(a->M >= 1 && a->N >= 1 && a->K >= 1, "gemm: empty problem %lldx%lldx%lld", (long long)a->M,
                  (long long)a->N, (long long)a->K);
  DIPPM_ARG_CHECK(a->a.dtype == a->b.dtype, "gemm: operand dtypes differ");
  cudaStream_t s = (cudaStream_t)stream;
  DIPPM_ARG_CHECK(!a->pool_partial || backend == 0, "gemm: the fused readout is a tensor-core epilogue");
  if (backend == 1) return dippm_gemm_simt_impl(a, s);
  DIPPM_ARG_CHECK(a->a.dtype == DIPPM_DT_BF16 || a->a.dtype == DIPPM_DT_TF32X3,
                  "gemm: tensor-core path needs bf16 or tf32x3 operands");
  DIPPM_ARG_CHECK(a->N % 64 == 0, "gemm: N=%lld must be a multiple of 64", (long long)a->N);
  DIPPM_ARG_CHECK(a->kind >= DIPPM_GEMM_FWD && a->kind <= DIPPM_GEMM_GATE, "gemm: bad kind %lld",
                  (long long)a->kind);
  const bool mn = a->kind == DIPPM_GEMM_WGRAD;
  DIPPM_ARG_CHECK(mn == (a->a_mn_major != 0) && (mn == (a->b_mn_major != 0) || a->kind == DIPPM_GEMM_FWD),
                  "gemm: FWD takes K-major A (B either), STORE/GATE K-major, WGRAD MN-major");
  DIPPM_ARG_CHECK(!a->pool_partial || (a->kind == DIPPM_GEMM_FWD && a->pool_graph && a->node_graph && a->graph_ptr),
                  "gemm: the fused readout needs FWD on the tensor-core backend with pool_graph, node_graph, graph_ptr");
  DIPPM_ARG_CHECK(a->out.data || a->pool_partial || a->kind == DIPPM_GEMM_STORE || a->kind == DIPPM_GEMM_WGRAD,
                  "gemm: FWD/GATE need an output view");
  DIPPM_ARG_CHECK(a->drop_mode == 0 || ((a->mask || a->drop_mode == 2) && a->kind == DIPPM_GEMM_FWD &&
                                        a->b_mn_major && a->drop_p >= 0 && a->drop_p < 1 && a->ldm % 4 == 0),
                  "gemm: dropout needs FWD with MN-major B, 0 <= p < 1, ldm %% 4 == 0 and (mode 1) a mask buffer");
  const int bk = a->a.dtype == DIPPM_DT_BF16 ? 64 : 32;
  DIPPM_ARG_CHECK(mn || a->K % bk == 0, "gemm: K=%lld must be a multiple of %d", (long long)a->K, bk);
  if (tc::shortk_ok(a)) return tc::run_shortk(a, s);
  if (a->a.dtype == DIPPM_DT_BF16) return tc::dispatch<1>(a, s);
  return tc::dispatch<2>(a, s);
}

// Fixed-order split-K reduction with transpose: out[j*ldo + i] = scale * sum_s in[s][i][j].
__global__ void k_splitk_reduce_t(const float* __restrict__ in, int splits, int64_t M, int64_t N, double scale,
                                  float* __restrict__ out, int64_t ldo) {
  __shared__ float tile[32][33];
  const int64_t i0 = (int64_t)blockIdx.y * 32, j0 = (int64_t)blockIdx.x * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = i0 + r, j = j0 + threadIdx.x;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;  // 4 independent chains, combined in fixed order
    if (i < M && j < N) {
      const float* p = in + i * N + j;
      const int64_t st = M * N;
      int sp = 0;
      for (; sp + 3 < splits; sp += 4) {
        a0 += (double)p[sp * st];
        a1 += (double)p[(sp + 1) * st];
        a2 += (double)p[(sp + 2) * st];
        a3 += (double)p[(sp + 3) * st];
      }
      for (; sp < splits; ++sp) a0 += (double)p[sp * st];
    }
    tile[r][threadIdx.x] = (float)(((a0 + a1) + (a2 + a3)) * scale);
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t j = j0 + r, i = i0 + threadIdx.x;
    if (i < M && j < N) out[j * ldo + i] = tile[threadIdx.x][r];
  }
}

extern "C" int32_t dippm_splitk_reduce_t(const float* in, int32_t splits, int64_t M, int64_t N, double scale,
                                         float* out, int64_t ldo, void* stream) {
  DIPPM_ARG_CHECK(splits >= 1 && M >= 1 && N >= 1, "splitk_reduce_t: bad shape");
  dim3 grid(ceil_div_i(N, 32), ceil_div_i(M, 32));
  k_splitk_reduce_t<<<grid, dim3(32, 8), 0, (cudaStream_t)stream>>>(in, splits, M, N, scale, out, ldo);
  DIPPM_LAUNCH_CHECK("k_splitk_reduce_t");
  return DIPPM_OK;
}
