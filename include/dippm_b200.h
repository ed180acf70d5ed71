/*
 * dippm_b200.h — C ABI of the B200-native DIPPM GraphSAGE hot path.
 *
 * The reference (DIPPM, arXiv 2303.11733; /root/reference/pkg/src/dippm) is a
 * pure-Python/numpy package with no native code, so there is no existing
 * plugin ABI to mirror.  These entry points are what a ctypes binding of the
 * reference's per-record numpy expressions would bind once they are batched
 * over many graphs; each declaration cites the reference expression it
 * replaces.  INTEGRATION.md shows the ctypes stubs.
 *
 * Conventions
 *  - plain pointers and sizes only; no torch / C++ types;
 *  - every pointer argument documented "device" is CUDA device memory, the
 *    caller owns it, the library never allocates or frees caller memory
 *    (kernels are therefore capturable in CUDA graphs);
 *  - `stream` is a cudaStream_t passed as void*; all work is stream-ordered,
 *    nothing synchronises the host unless the name says so;
 *  - return value: DIPPM_OK or an error code, with a message available from
 *    dippm_last_error() (thread-local).  The Python layer maps the codes onto
 *    the reference's DippmError hierarchy (errors.py:8-83).
 *  - node / edge indices in a batch are global (graph offsets applied), the
 *    batch is described by graph_ptr[G+1] (rows graph_ptr[g]..graph_ptr[g+1]).
 */
#ifndef DIPPM_B200_H_
#define DIPPM_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DIPPM_ABI_VERSION 1

enum dippm_status {
  DIPPM_OK = 0,
  DIPPM_ERR_ARG = 1,         /* bad argument (ShapeMismatch / ValueError in the reference) */
  DIPPM_ERR_CUDA = 2,        /* CUDA runtime / launch failure */
  DIPPM_ERR_NONFINITE = 3,   /* NaN/Inf where the reference raises NonFinite (mig.py:38-39) */
  DIPPM_ERR_UNSUPPORTED = 4  /* shape outside what the kernels support */
};

/* Element types of activation buffers. */
enum dippm_dtype {
  DIPPM_DT_F32 = 0,     /* plain fp32 */
  DIPPM_DT_BF16 = 1,    /* bf16 operands, fp32 accumulate (bf16 mode) */
  DIPPM_DT_TF32X3 = 2   /* fp32 stored as two fp32 planes hi/lo for the 3-pass tf32 split (fp32 mode) */
};

/* An activation matrix [rows, cols] with row stride ld (elements).  For
 * DIPPM_DT_TF32X3 the lo plane starts plane_stride elements after data. */
typedef struct dippm_act {
  void* data;
  int64_t ld;
  int64_t plane_stride;
  int64_t dtype;
} dippm_act_t;

const char* dippm_last_error(void);
int32_t dippm_abi_version(void);
/* Total kernel launches issued by this library since load (bench evidence). */
uint64_t dippm_launch_count(void);
/* Number of SMs of the current device (grid sizing; 148 on B200). */
int32_t dippm_device_sm_count(void);

/* ---------------------------------------------------------------------------
 * MIG profile pick — mig.py:32-45 (MigProfile ceilings mig.py:19-22).
 * code: 0=1g.5gb 1=2g.10gb 2=3g.20gb 3=7g.40gb, -1 = None.
 * The host and device implementations share one __host__ __device__ rule.  */
int32_t dippm_mig_code(double alpha_mb, int32_t* code);
/* Batched, on device: codes[g] from mem_mb[g*stride]; *nonfinite (device
 * int32) is set to 1 if any input is NaN/Inf (the caller raises NonFinite). */
int32_t dippm_mig_codes(const double* mem_mb, int64_t stride, int64_t count, int8_t* codes,
                        int32_t* nonfinite, void* stream);

/* ---------------------------------------------------------------------------
 * K1 — CSR construction.  Replaces _aggregation_matrix gnn.py:130-137 (and
 * its transpose, used at gnn.py:161-162).
 *   rows = dst, cols = distinct src of the row, ascending (deterministic);
 *   deg[v] = in-degree counting duplicate edges (gnn.py:133-134);
 *   inv_deg[v] = 1/deg[v] or 0 (isolated, gnn.py:131 zero row);
 *   t_rowptr/t_col: the transposed pattern (rows = src, cols = dst ascending).
 * src/dst: device int64 [E]; rowptr/t_rowptr: device int32 [N+1];
 * col/t_col: device int32 [E] (capacity; rowptr[N] holds the unique count);
 * bad_edge: device int32, set to 1 if an endpoint is outside [0, N). */
size_t dippm_csr_workspace_bytes(int64_t num_nodes, int64_t num_edges);
int32_t dippm_build_csr(const int64_t* src, const int64_t* dst, int64_t num_edges, int64_t num_nodes,
                        int32_t* rowptr, int32_t* col, int32_t* deg, float* inv_deg,
                        int32_t* t_rowptr, int32_t* t_col, int32_t* bad_edge,
                        void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * K2 — neighbour mean m = agg @ h (gnn.py:157-158 via _embed gnn.py:206).
 * h: [N, width] activation view; m_out: [N, width] view (usually the right
 * half of the layer's [h | m] GEMM operand).  If self_out.data is non-NULL
 * the kernel also copies h into it (layer-1 operand assembly).  width % 8 == 0. */
int32_t dippm_sage_aggregate(dippm_act_t h, dippm_act_t m_out, dippm_act_t self_out, int64_t num_nodes,
                             int32_t width, const int32_t* rowptr, const int32_t* col,
                             const float* inv_deg, void* stream);

/* K2 backward — gnn.py:227,232: given dA = dz @ [W_self; W_neigh]^T as fp32
 * [N, 2*width] (row stride ld_da), computes
 *   dh[u]  = dA[u, :width] + sum_{v in out(u)} inv_deg[v] * dA[v, width:]
 *   dz[u]  = dh[u] * (h_prev[u] > 0)          (ReLU mask of the layer below)
 * writes dz into dz_out, and per-block column partial sums of dz into
 * colsum_partial [dippm_colsum_blocks(N), width] (bias gradient, gnn.py:230,
 * reduced deterministically by dippm_reduce_rows). */
int32_t dippm_colsum_blocks(int64_t num_nodes);
int32_t dippm_sage_backward_gather(const float* dA, int64_t ld_da, int32_t width, dippm_act_t h_prev,
                                   dippm_act_t dz_out, int64_t num_nodes, const int32_t* t_rowptr,
                                   const int32_t* t_col, const float* inv_deg, float* colsum_partial,
                                   void* stream);

/* Readout backward — gnn.py:224,227: dz3[v] = dr[g(v)] / N_g * (h3[v] > 0),
 * dr = du[:, :width] with du [G, ld_du] fp32; plus column partial sums. */
int32_t dippm_readout_backward(const float* du, int64_t ld_du, const int32_t* graph_ptr, int64_t num_graphs,
                               int32_t width, dippm_act_t h3, dippm_act_t dz_out, int64_t num_nodes,
                               float* colsum_partial, void* stream);

/* out[c] = scale * sum_{r<rows} in[r*ld + c] in fixed row order (fp32 in, fp64 accumulate). */
int32_t dippm_reduce_rows(const float* in, int64_t rows, int64_t ld, int32_t cols, double scale,
                          float* out, void* stream);

/* ---------------------------------------------------------------------------
 * K3 — GEMMs on the 5th-gen tensor cores (tcgen05 + TMEM + TMA), or the SIMT
 * fp32 kernel (backend 1, a parity anchor for tests).
 *   FWD:    out = act(A @ B^T + bias)   A [M,K] (= [h | m]), B [N,K] packed W^T
 *           — gnn.py:207-209 (z = h@W_self + m@W_neigh + bias; h = relu(z))
 *   STORE:  C[M,N] fp32 = A @ B^T        — dgrad, gnn.py:232 (dz @ W^T)
 *   WGRAD:  C_s[M,N] fp32 partials of A^T-style products with both operands
 *           MN-major: C = dz^T @ [h | m] split over row chunks s — gnn.py:228-229
 * Operand "major": 0 = K-major ([rows, K] row-major), 1 = MN-major ([K, rows]). */
enum dippm_gemm_kind { DIPPM_GEMM_FWD = 0, DIPPM_GEMM_STORE = 1, DIPPM_GEMM_WGRAD = 2 };

typedef struct dippm_gemm_args {
  int64_t kind;
  int64_t M, N, K;
  dippm_act_t a;       /* dtype BF16 or TF32X3 (both operands the same dtype) */
  int64_t a_mn_major;
  dippm_act_t b;
  int64_t b_mn_major;
  const float* bias;   /* FWD: [N] fp32 */
  int64_t relu;        /* FWD */
  dippm_act_t out;     /* FWD output view */
  float* c;            /* STORE: [M, ldc]; WGRAD: [splits, M, ldc] */
  int64_t ldc;
  int64_t splits;      /* WGRAD split count (>=1); others 1 */
} dippm_gemm_args_t;

/* Split count the tensor-core WGRAD would like for this problem. */
int32_t dippm_wgrad_splits(int64_t M, int64_t N, int64_t K);
int32_t dippm_gemm(const dippm_gemm_args_t* args, int32_t backend, void* stream);

/* out[j*ldo + i] = scale * sum_s in[s*M*N + i*N + j]  (split-K reduce + transpose; fixed order) */
int32_t dippm_splitk_reduce_t(const float* in, int32_t splits, int64_t M, int64_t N, double scale, float* out,
                              int64_t ldo, void* stream);

/* ---------------------------------------------------------------------------
 * K4 — readout + static features: u[g] = [ mean_{v in g} h3[v] , (fs[g]-fs_mean)/fs_std ]
 * gnn.py:214-215, normalize_fs gnn.py:96-97.  u: [G, width+5] fp32.
 * norm: device double[16] = y_mean[3], y_std[3], fs_mean[5], fs_std[5]. */
int32_t dippm_pool_concat(dippm_act_t h, const int32_t* graph_ptr, int64_t num_graphs, int32_t width,
                          const float* fs_raw, const double* norm, float* u, void* stream);

/* ---------------------------------------------------------------------------
 * K5 — FC head, gnn.py:265-284: fc1 (width+5 -> width) ReLU (+dropout),
 * fc2 (width -> width) ReLU (+dropout), fc3 (width -> 3).
 * head_w: device fp32, packed [fc1.w (width+5)*width | fc1.b | fc2.w | fc2.b | fc3.w | fc3.b].
 * cache: device fp32 [4, G, width] = a1, x2, a2, x3 (pre-activations and layer inputs).
 * masks: device fp32 [2, G, width]; mask_mode 0 = none (eval), 1 = use given
 * masks (host-drawn PCG64, numerics.py:45-55), 2 = generate (counter hash, seed).
 * out_norm: [G,3] fp32 normalised outputs.  If y_pred (device double [G,3]) is
 * non-NULL, also de-normalises (gnn.py:93-94) and writes MIG codes
 * (mig.py:32-45) from y_pred[:,1] into mig (int8 [G]). */
int32_t dippm_head_forward(const float* u, int64_t num_graphs, int32_t width, const float* head_w,
                           float* cache, float* masks, int32_t mask_mode, float dropout_p, uint64_t seed,
                           float* out_norm, const double* norm, double* y_pred, int8_t* mig,
                           int32_t* nonfinite, void* stream);

/* Huber loss + gradient, numerics.py:58-73, averaged over the batch
 * (gnn.py:398-404): dout[g] = grad_g / G.  y_raw [G,3] fp32 targets are
 * normalised on device (gnn.py:90-91).  loss_out: device double [4] =
 * {mean loss, sum APE latency, memory, energy} (APE uses de-normalised
 * outputs, gnn.py:458-459). */
int32_t dippm_huber(const float* out_norm, const float* y_raw, int64_t num_graphs, const double* norm,
                    double delta, float* dout, double* loss_out, void* stream);

/* Head backward, gnn.py:287-299: writes fc grads into grads_head (same
 * packing as head_w) and du [G, width+5] fp32 (input gradient). */
int32_t dippm_head_backward(const float* u, int64_t num_graphs, int32_t width, const float* head_w,
                            const float* cache, const float* masks, int32_t use_masks, const float* dout,
                            float* grads_head, float* du, float* scratch, void* stream);
size_t dippm_head_scratch_floats(int64_t num_graphs, int32_t width);

/* ---------------------------------------------------------------------------
 * K8 — bias-corrected Adam, numerics.py:93-114, same op order, on fp64
 * master parameters (fp32 gradients, multiplied by grad_scale first — 1/world
 * size after a data-parallel sum), one launch for all 15 tensors. */
int32_t dippm_adam(double* params, double* m, double* v, const float* grads, double grad_scale, int64_t n,
                   int64_t t, double lr, double beta1, double beta2, double eps, void* stream);

/* Pack fp64 master weights into compute copies.
 *  w [rows, cols] fp64 row-major  ->  dst view (bf16 or tf32 hi/lo or f32);
 *  transpose != 0 writes dst[c, r] (K-major W^T for the forward GEMM). */
int32_t dippm_pack(const double* w, int64_t rows, int64_t cols, int32_t transpose, dippm_act_t dst, void* stream);

/* Batch assembly from a device-resident dataset (bench / training epochs):
 * gathers graphs ids[0..G) into contiguous rows. */
int32_t dippm_gather_rows(const float* src, const int64_t* src_row, int64_t rows, int32_t cols, float* dst,
                          void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DIPPM_B200_H_ */
