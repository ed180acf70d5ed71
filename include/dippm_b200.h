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

#define DIPPM_ABI_VERSION 15

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
/* Grouped fast path (same outputs, bit for bit): the batch is a concatenation of
 * graphs — graph_ptr [G+1] over nodes, edge_ptr [G+1] over edges (int64), every
 * edge inside its own graph (else *bad_edge = 1).  One CTA per graph builds its
 * CSR in shared memory and finds its offset in the packed arrays by a decoupled look-back
 * (one memset + one launch per batch; the workspace holds the per-graph status words).
 * Limits: G <= 8192, per-graph edges and nodes <= 8192; callers fall back to
 * dippm_build_csr beyond.
 * node_graph (nullable): also writes the node -> graph map (dippm_node_graph) in the same pass. */
size_t dippm_csr_grouped_workspace_bytes(int64_t num_graphs, int64_t num_edges);
/* The same, fused with the layer-1 operand of the training step (gnn.py:157-158 for the fp32
 * 32-wide input x [N, 32]): a1[v, 0:32] = bf16(x[v]), a1[v, 32:64] = bf16(inv_deg[v] * sum over
 * v's in-neighbours of x, CSR order) -- dippm_sage_aggregate's result bit for bit, without its
 * launch.  a1: bf16 view, ld >= 64 (columns >= 64 untouched). */
int32_t dippm_build_csr_grouped_l1(const int64_t* src, const int64_t* dst, const int32_t* graph_ptr,
                                   const int64_t* edge_ptr, int64_t num_graphs, int64_t num_nodes, int64_t num_edges,
                                   int32_t max_nodes_per_graph, int32_t max_edges_per_graph, int32_t* rowptr,
                                   int32_t* col, int32_t* deg, float* inv_deg, int32_t* t_rowptr, int32_t* t_col,
                                   int32_t* bad_edge, int32_t* node_graph, void* workspace, size_t workspace_bytes,
                                   const float* x, dippm_act_t a1, void* stream);
int32_t dippm_build_csr_grouped(const int64_t* src, const int64_t* dst, const int32_t* graph_ptr,
                                const int64_t* edge_ptr, int64_t num_graphs, int64_t num_nodes, int64_t num_edges,
                                int32_t max_nodes_per_graph, int32_t max_edges_per_graph,
                                int32_t* rowptr, int32_t* col, int32_t* deg, float* inv_deg,
                                int32_t* t_rowptr, int32_t* t_col, int32_t* bad_edge, int32_t* node_graph,
                                void* workspace, size_t workspace_bytes, void* stream);
int32_t dippm_build_csr(const int64_t* src, const int64_t* dst, int64_t num_edges, int64_t num_nodes,
                        int32_t* rowptr, int32_t* col, int32_t* deg, float* inv_deg,
                        int32_t* t_rowptr, int32_t* t_col, int32_t* bad_edge,
                        void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * K2 — neighbour mean m = agg @ h (gnn.py:157-158 via _embed gnn.py:206).
 * h: [N, width] activation view; m_out: [N, width] view (usually the right
 * half of the layer's [h | m] GEMM operand).  If self_out.data is non-NULL
 * the kernel also copies h into it (layer-1 operand assembly).  width: 8 * 2^k (8..1024) or 24 * 2^k (24..768) columns -- the
 * 8-column chunks of a row must tile a warp (three per lane for the 3 * 2^k widths). */
int32_t dippm_sage_aggregate(dippm_act_t h, dippm_act_t m_out, dippm_act_t self_out, int64_t num_nodes,
                             int32_t width, const int32_t* rowptr, const int32_t* col,
                             const float* inv_deg, void* stream);

/* K2 backward — gnn.py:161-162, 227-232.  B = [dz | g] is [N, 2*width]
 * (row stride B.ld) with dz in the left half; writes g = agg^T dz into the
 * right half (g[u] = sum_{u->v} dz[v] / deg v, via the transposed CSR), so the
 * input gradient dh_prev = [dz | g] @ [W_self | W_neigh]^T is one GATE GEMM.
 * Also reduces the columns of dz (bias gradient gnn.py:230): per-block partial
 * sums go to colsum_partial [dippm_colsum_rows(N), width]; with bias_grad !=
 * NULL the kernel finishes the reduction itself (two fixed-order levels, last
 * block of each group / last group, fp64 sums) and writes bias_grad [width];
 * sync is device int32[dippm_colsum_sync_ints(N)], zeroed once by the caller
 * and left zero by every launch.  With bias_grad == NULL and sync == NULL only the first
 * dippm_colsum_blocks(N) partial rows are written (reduce with dippm_reduce_rows).  With
 * bias_grad == NULL and sync != NULL (deferred fold) the kernel keeps its wave-sized blocks,
 * writes their partial rows and their count (int32 at dippm_colsum_count_slot) for the
 * layer's weight-gradient GEMM to fold (dippm_gemm_args_t.bias_partial).
 * write_agg = 0 computes the column sums only. */
int32_t dippm_colsum_blocks(int64_t num_nodes);
int32_t* dippm_colsum_count_slot(float* colsum_partial, int64_t num_nodes, int32_t width);
int32_t dippm_colsum_rows(int64_t num_nodes);
int32_t dippm_colsum_sync_ints(int64_t num_nodes);
int32_t dippm_sage_aggregate_t(dippm_act_t B, int32_t width, int64_t num_nodes, int32_t write_agg,
                               const int32_t* t_rowptr, const int32_t* t_col, const float* inv_deg,
                               float* colsum_partial, float* bias_grad, int32_t* sync, void* stream);

/* Layer-3 variant with the readout backward fused in (gnn.py:224, 227): dz3 is
 * formed on the fly as dz3[v] = du[g(v), :width] / N_g * (h3[v] > 0), written to
 * B's left half, while agg^T dz3 goes to the right half and the bias partial
 * sums to colsum_partial.  node_graph [N] maps node -> graph (dippm_node_graph). */
int32_t dippm_readout_aggregate_t(const float* du, int64_t ld_du, const int32_t* graph_ptr,
                                  const int32_t* node_graph, dippm_act_t h3, dippm_act_t B, int32_t width,
                                  int64_t num_nodes, const int32_t* t_rowptr, const int32_t* t_col,
                                  const float* inv_deg, float* colsum_partial, float* bias_grad, int32_t* sync,
                                  const uint32_t* h3_bits, int64_t bits_ld, void* stream);
/*   h3_bits (optional): the layer-3 forward GEMM's 1-bit (h3 > 0) masks (dippm_gemm relu_bits
 *   layout: chunk-major with bits_ld >= N, or row-major with bits_ld == 0 -- the layout this
 *   kernel reads best, one row's words being contiguous); used instead of reading h3. */
/* node_graph[v] = g for v in [graph_ptr[g], graph_ptr[g+1]). */
int32_t dippm_node_graph(const int32_t* graph_ptr, int64_t num_graphs, int32_t* node_graph, void* stream);

/* Readout backward alone — gnn.py:224,227: dz3[v] = du[g(v), :width] / N_g * (h3[v] > 0),
 * du [G, ld_du] fp32. */
int32_t dippm_readout_backward(const float* du, int64_t ld_du, const int32_t* graph_ptr, int64_t num_graphs,
                               int32_t width, dippm_act_t h3, dippm_act_t dz_out, int64_t num_nodes, void* stream);

/* out[c] = scale * sum_{r<rows} in[r*ld + c] in fixed row order (fp32 in, fp64 accumulate). */
int32_t dippm_reduce_rows(const float* in, int64_t rows, int64_t ld, int32_t cols, double scale,
                          float* out, void* stream);

/* ---------------------------------------------------------------------------
 * K3 — GEMMs on the 5th-gen tensor cores (tcgen05 + TMEM + TMA), or the SIMT
 * fp32 kernel (backend 1, a parity anchor for tests).
 *   FWD:    out = act(A @ B^T + bias)   A [M,K] (= [h | m]), B [N,K] packed W^T
 *           — gnn.py:207-209 (z = h@W_self + m@W_neigh + bias; h = relu(z))
 *   STORE:  C[M,N] fp32 = A @ B^T        — dgrad, gnn.py:232 (dz @ W^T)
 *   WGRAD:  C[M,N] fp32 = A^T-style product with both operands MN-major, the reduction
 *           (over node rows) split in `splits` chunks — gnn.py:228-229
 *           ([h | m]^T @ dz = [dW_self; dW_neigh]).  With tile_sync != NULL the kernel
 *           reduces the split partials itself (fixed split order, fp64 sums, see
 *           tile_sync) and writes out = out_scale * C into `out` (F32 view); with
 *           tile_sync == NULL it only writes the partials C_s to c.
 * Operand "major": 0 = K-major ([rows, K] row-major), 1 = MN-major ([K, rows]). */
enum dippm_gemm_kind { DIPPM_GEMM_FWD = 0, DIPPM_GEMM_STORE = 1, DIPPM_GEMM_WGRAD = 2, DIPPM_GEMM_GATE = 3 };
/*   GATE:   out = (gate > 0) * gate_scale * (A @ B^T)  — dgrad fused with the ReLU (+dropout)
 *           mask of the layer below: gnn.py:227,232 / 293-298, A = [dz | agg^T dz].          */

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
  float* c;            /* STORE: [M, ldc]; WGRAD: [splits, M, ldc] partials (unused if splits == 1 and fused) */
  int64_t ldc;
  int64_t splits;      /* WGRAD split count (>=1); others 1 */
  dippm_act_t gate;    /* GATE: out = gate > 0 ? acc * gate_scale : 0 (ReLU' of the layer below, */
  double gate_scale;   /*       times the inverted-dropout keep scale where one applies)          */
  int64_t drop_mode;   /* FWD dropout after ReLU: 0 none, 1 multiply mask, 2 generate mask (hash) */
  float* mask;         /* [M, ldm] fp32 dropout mask (read in mode 1, written in mode 2)         */
  int64_t ldm;
  double drop_p;
  uint64_t seed;
  const int64_t* seed_dev; /* nullable device step counter mixed into the dropout seed (graph replays) */
  uint32_t* relu_bits;       /* FWD (optional): bit c%32 of word [(c/32)*bits_ld + r] = (stored out[r,c] > 0); */
                             /* bits_ld == 0: row-major instead, word [r*(N/32) + c/32] (FWD relu_bits only)  */
  const uint32_t* gate_bits; /* GATE (optional): use these bits instead of reading `gate` values          */
                             /* (relu_bits / gate_bits: tensor-core backend; the SIMT anchor gates on values) */
  int64_t bits_ld;           /* words per 32-column chunk of relu_bits / gate_bits (chunk-major, >= M)   */
  int64_t cta_pair;          /* 0 auto, 1 force 1-CTA 128-row tiles, 2 force cta_group::2 256-row tiles   */
  int32_t* tile_sync;        /* WGRAD fused reduce: device int32[dippm_wgrad_sync_ints(M, N)], zeroed once  */
                             /* by the caller; every launch leaves it zero again (graph-replay safe)      */
  double out_scale;          /* WGRAD fused reduce: out = out_scale * sum_s C_s                            */
  /* FWD with the K4 readout fused into the epilogue (gnn.py:214, rows = nodes, N = width):
   * per 32-row block, a segmented (by graph) column sum of the stored activation goes to
   * pool_graph [G, N] (graphs wholly inside the block) or to pool_partial [2*ceil(M/32), N]
   * (slot 0: the block's first graph, slot 1: its last, when they cross the block edge);
   * dippm_pool_combine then forms the means.  out.data may be NULL (the activation itself is
   * not needed).  Tensor-core backend only. */
  float* pool_partial;
  float* pool_graph;
  const int32_t* node_graph;   /* [M] node -> graph */
  const int32_t* graph_ptr;    /* [G+1] */
  /* WGRAD (optional): also fold the layer's bias gradient, bias_grad[N] = column sums of the
   * partial rows an agg^T / readout kernel left in deferred mode (bias_grad NULL, sync given)
   * in bias_partial ([dippm_colsum_rows(K), N]; K = the rows reduced = the layer's nodes).  The
   * fold rides in the weight-gradient launch (off the dgrad chain) instead of the tail of the
   * aggregation kernel. */
  const float* bias_partial;
  float* bias_grad;
} dippm_gemm_args_t;

/* Split count the tensor-core WGRAD would like for this problem. */
int32_t dippm_wgrad_splits(int64_t M, int64_t N, int64_t K);
/* Size (int32 elements) of the WGRAD tile_sync counter array for an M x N output. */
int64_t dippm_wgrad_sync_ints(int64_t M, int64_t N);
int32_t dippm_gemm(const dippm_gemm_args_t* args, int32_t backend, void* stream);

/* out[j*ldo + i] = scale * sum_s in[s*M*N + i*N + j]  (split-K reduce + transpose; fixed order) */
int32_t dippm_splitk_reduce_t(const float* in, int32_t splits, int64_t M, int64_t N, double scale, float* out,
                              int64_t ldo, void* stream);

/* K4 second stage of the fused readout: u[g] = [ (sum of g's block sums, fixed block
 * order) / N_g , (fs[g] - fs_mean) / fs_std , 0 ... ] from the FWD epilogue's pool_partial /
 * pool_graph (see dippm_gemm_args_t).  dippm_pool_partial_rows(N) = rows of pool_partial. */
int64_t dippm_pool_partial_rows(int64_t num_nodes);
int32_t dippm_pool_combine(const float* pool_partial, const float* pool_graph, const int32_t* graph_ptr,
                           int64_t num_graphs, int32_t width, const double* fs_raw, const double* norm, dippm_act_t u,
                           void* stream);

/* ---------------------------------------------------------------------------
 * K4 — readout + static features (gnn.py:214-215, normalize_fs gnn.py:96-97):
 *   u[g] = [ mean_{v in g} h3[v] , (fs[g] - fs_mean) / fs_std , 0 ... ]
 * u: [G, u.ld] activation view in the head's operand dtype, u.ld >= width + 5
 * (zero padded so fc1 runs as a K-aligned tensor-core GEMM).
 * norm: device double[16] = y_mean[3], y_std[3], fs_mean[5], fs_std[5]. */
int32_t dippm_pool_concat(dippm_act_t h, const int32_t* graph_ptr, int64_t num_graphs, int32_t width,
                          const double* fs_raw, const double* norm, dippm_act_t u, void* stream);

/* MLP baseline input (MlpModel.forward_norm gnn.py:253-255, normalize_fs gnn.py:96-97):
 * u[g, c] = (fs_raw[g, c] - fs_mean[c]) / fs_std[c] for c < 5, 0 for 5 <= c < cols. */
int32_t dippm_fs_normalize(const double* fs_raw, int64_t num_graphs, const double* norm, dippm_act_t u,
                           int32_t cols, void* stream);

/* ---------------------------------------------------------------------------
 * K5 — FC head, gnn.py:265-284.  fc1/fc2 (and their gradients) are dippm_gemm
 * calls: FWD with bias + ReLU + dropout epilogue, GATE / STORE / WGRAD for the
 * backward.  fc3 (width -> 3) and the output stage are:
 * dippm_fc3_forward: out_norm[g] = x3[g] @ w3 + b3 (normalised, [G,3] fp32);
 * if y_pred != NULL also de-normalises (gnn.py:93-94, fp64) and writes the
 * MIG code of y_pred[g,1] (mig.py:32-45) into mig[g]; *nonfinite set on NaN/Inf. */
int32_t dippm_fc3_forward(dippm_act_t x3, int64_t num_graphs, int32_t width, const float* w3, const float* b3,
                          float* out_norm, const double* norm, double* y_pred, int8_t* mig, int32_t* nonfinite,
                          void* stream);

/* fc3 backward fused with the fc2 ReLU/dropout gate (gnn.py:293-298):
 *   grad_w3 = x3^T dout, grad_b3 = sum dout, d2 = (dout @ w3^T) * (x3 > 0) * keep_scale,
 *   grad_b2 = column sums of d2.  keep_scale = 1/(1-p) in train mode with dropout, else 1. */
int32_t dippm_fc3_backward(dippm_act_t x3, int64_t num_graphs, int32_t width, const float* w3, const float* dout,
                           float keep_scale, float* grad_w3, float* grad_b3, dippm_act_t d2, float* grad_b2,
                           void* stream);

/* Column sums of an activation view (fixed order): out[c] = sum_r a[r, c]. */
int32_t dippm_colsum_act(dippm_act_t a, int64_t rows, int32_t cols, float* out, void* stream);

/* Huber loss + gradient, numerics.py:58-73, averaged over the batch
 * (gnn.py:398-404): dout[g] = grad_g / G (dout may be NULL).  y_raw [G,3] fp64
 * targets are normalised on device (gnn.py:90-91).  loss_out: device double[4]
 * = {mean loss, sum APE latency, memory, energy} (APE on de-normalised
 * outputs, gnn.py:458-459). */
int32_t dippm_huber(const float* out_norm, const double* y_raw, int64_t num_graphs, const double* norm,
                    double delta, double grad_den, float* dout, double* loss_out, void* stream);
/*   grad_den: denominator of dout (<= 0: num_graphs).  Data-parallel training passes the
 *   GLOBAL batch size so the all-reduced sum of per-rank gradients is the global mean. */

/* ---------------------------------------------------------------------------
 * K5/K6 fused — the whole FC head of one step in ONE cooperative launch (bf16, small
 * batches: 1 <= G <= dippm_head_fused_max_graphs(), hp % 64 == 0, hp <= 512, u_width a
 * multiple of 64 <= 576).  Replaces, for those shapes, the fc1/fc2 dippm_gemm calls,
 * dippm_fc3_forward, dippm_huber, dippm_fc3_backward, dippm_colsum_act and the fc2/fc1
 * WGRAD / GATE / STORE GEMMs (gnn.py:265-299, numerics.py:58-73):
 *   always    x2 = drop1(relu(u W1 + b1)), x3 = drop2(relu(x2 W2 + b2)) (bf16 [G, hp]),
 *             out = x3 W3 + b3 (normalised fp32 [G, 3]); bits (if non-NULL) = x2 > 0,
 *             word [(c/32)*bits_ld + g]; y_pred / mig / nonfinite as dippm_fc3_forward.
 *   y_raw     Huber per graph, loss_out = {mean loss, APE sums} as dippm_huber, dout.
 *   train     d2 = (dout W3^T)[x3 > 0] keep, d1 = (d2 W2^T)[x2 > 0] keep (bf16 + fp32
 *             copies), gw3/gb3/gw2/gb2/gw1/gb1 (fp32, padded layouts [hp,3], [hp,hp],
 *             [u_width,hp]) and, if du != NULL, du = d1 W1[:hp]^T (fp32 [G, hp]).
 * Dropout: mode 0 none, 1 multiply mask1/mask2 ([G, hp] fp32), 2 the counter hash of
 * dippm_gemm (seed1/seed2, seed_dev mixed in identically), so the draws match that path.
 * sync: int32[dippm_head_fused_sync_ints()] zeroed once by the caller; left ready for the next
 * launch.
 * Every reduction has a fixed order (deterministic). */
typedef struct dippm_head_args {
  int64_t G;
  int32_t hp, u_width;
  const void* u;                 /* bf16 [G, u_width] */
  const void* w1;                /* bf16 [u_width, hp] */
  const void* w2;                /* bf16 [hp, hp] */
  const float *b1, *b2, *w3, *b3;/* fp32 [hp], [hp], [hp, 3], [3] */
  void *x2, *x3;                 /* bf16 [G, hp] (written) */
  uint32_t* bits;                /* word [(c/32)*bits_ld + g], or NULL */
  int64_t bits_ld;               /* >= G */
  int32_t drop_mode;
  double drop_p;
  float keep_scale;              /* backward gate scale: 1/(1-p) with dropout, else 1 */
  uint64_t seed1, seed2;
  const int64_t* seed_dev;
  const float *mask1, *mask2;
  float* out;                    /* fp32 [G, 3] */
  const double* norm;            /* double[16] as dippm_pool_concat */
  double* y_pred;                /* [G, 3] or NULL */
  int8_t* mig;
  int32_t* nonfinite;
  const double* y_raw;           /* [G, 3] fp64 targets or NULL (no loss) */
  double delta, grad_den;
  double* loss_out;              /* double[4] */
  double* row_loss;              /* scratch double [G, 4] */
  float* dout;                   /* [G, 3] (train) */
  void *d2, *d1;                 /* bf16 [G, hp] */
  float *d2f, *d1f;              /* fp32 [G, hp] */
  float *gw1, *gb1, *gw2, *gb2, *gw3, *gb3; /* gw1 / gw2 may be NULL in training: the caller then
                                    computes dW1 = u^T d1 and dW2 = x2^T d2 itself from the bf16 d1 /
                                    d2 this launch writes (off the critical path: dippm_train_step runs
                                    them as weight-gradient GEMMs on its side stream) */
  float* du;                     /* fp32 [G, hp] or NULL (MLP: no readout below) */
  int32_t* sync;
  int32_t train;
  /* optional (all four or none): u's readout columns are formed in-kernel from the layer-3
   * FWD epilogue's block sums, exactly as dippm_pool_combine does (then u is written, not read
   * from a separate launch); fs_raw [G, 5] fp64. */
  const float* pool_partial;
  const float* pool_graph;
  const int32_t* graph_ptr;
  const double* fs_raw;
  /* optional (training): step_counter[0] += 1 once every CTA is past the forward's dropout
   * draws (which read it through seed_dev) -- dippm_step_counter folded into this launch. */
  int64_t* step_counter;
  /* training: 1 leaves the column sums (db1, db2, dW3) and the batch loss + db3 to
   * dippm_head_reduce, launched after this kernel (the training step runs it on its side stream:
   * phases D / E then hold only what the readout backward waits for) */
  int32_t defer_reduce;
} dippm_head_args_t;
/* The reductions a defer_reduce head left: db2 + dW3, db1, loss_out + db3 (same units, same
 * results as inside the head kernel); stream-ordered after that head launch. */
int32_t dippm_head_reduce(const dippm_head_args_t* h, void* stream);
int32_t dippm_head_fused_max_graphs(void);
int32_t dippm_head_fused_sync_ints(void);
/* Opt-in tensor-core head: training-step heads with G <= 256, hp == 512, u_width == 576 (and no
 * phase 0 / predict / mask-mode dropout) on one cluster of 8 CTAs, tcgen05 + TMA + TMEM
 * (head_tc.cu; ~4x slower than the default 148-CTA kernel at configs[1], kept as the tested
 * tcgen05 formulation).  on = 0 / 1 switches it off / on (on < 0: query); returns the previous
 * state.  Also DIPPM_HEAD_TC=1 at load. */
int32_t dippm_head_tc_enable(int32_t on);
/* Diagnostics (synchronous): globaltimer stamps of CTA 0 of the last tensor-core head launch:
 * kernel start (after setup) and the end of each of its 8 phases (P1 P2 C D P3 P4 P5 P6). */
int32_t dippm_head_tc_trace(uint64_t* out16);
int32_t dippm_head_fused(const dippm_head_args_t* args, void* stream);
/* Diagnostics (synchronous): SM clock cycles, relative to kernel start, of CTA 0 of the last
 * launch: per phase (A, B: slots 1-4 / 5-8; C ends at 9, barrier 10; D 11-14; E 15-18) its
 * first unit's operands landed, that unit done, its last unit done, the grid barrier opened. */
int32_t dippm_head_fused_trace(int64_t* out24);

/* ---------------------------------------------------------------------------
 * K8 — bias-corrected Adam (numerics.py:93-114, same op order) on fp64 master
 * parameters, fused with the refresh of every compute copy the GEMMs read.
 * grads (fp32) are multiplied by grad_scale first (1/world after a data-
 * parallel sum).  do_adam = 0 only refreshes the copies.  p32 (fp32 [n]) gets
 * the updated parameters; each segment copies params[src_off .. + rows*cols)
 * (row-major [rows, cols]) into dst at (r, dst_col_off + c) in dst's dtype
 * (bf16, or tf32 hi/lo planes).  One launch for all 15 tensors. */
#define DIPPM_MAX_PACK_SEGS 12
typedef struct dippm_pack_seg {
  int64_t src_off;
  int64_t rows, cols;
  int64_t dst_col_off;
  dippm_act_t dst;
} dippm_pack_seg_t;
int32_t dippm_adam_pack(double* params, double* m, double* v, const float* grads, double grad_scale, int64_t n,
                        int64_t t, const int64_t* t_dev, double lr, double beta1, double beta2, double eps,
                        int32_t do_adam, float* p32, const dippm_pack_seg_t* segs, int32_t nsegs, void* stream);
/*   t_dev (nullable): device step counter; when given it overrides t (CUDA-graph replays). */
/* t_dev[0] += 1 on the stream (the per-step counter a captured training step replays). */
int32_t dippm_step_counter(int64_t* t_dev, void* stream);

/* Pack a fp64 matrix into a compute copy (tests / single-layer API):
 *  w [rows, cols] fp64 row-major -> dst view; transpose != 0 writes dst[c, r]. */
int32_t dippm_pack(const double* w, int64_t rows, int64_t cols, int32_t transpose, dippm_act_t dst, void* stream);

/* ---------------------------------------------------------------------------
 * fp64 numerics of the drop-in `numerics` module (numerics.py:23-114), bit-exact
 * with numpy for the element-wise operations (no FMA contraction, same operation
 * order) and for the Huber mean (numpy's pairwise summation order).
 *
 * numerics.py:58-73 huber_loss over n >= 1 elements: grad[i] = dL/dpred[i], elems[i]
 * the per-element loss (scratch, n doubles), loss[0] = mean.  Two launches. */
int32_t dippm_huber_f64(const double* pred, const double* target, int64_t n, double delta, double* grad,
                        double* elems, double* loss, void* stream);
/* numerics.py:93-114 adam_step on n elements: m, v updated in place, param_out = new value
 * (may alias param).  The scalars one_minus_beta{1,2} = 1 - beta and bias_corr{1,2} =
 * 1 - beta**t are passed from the host exactly as the reference computes them. */
int32_t dippm_adam(const double* param, const double* grad, double* m, double* v, double* param_out, int64_t n,
                   double lr, double beta1, double beta2, double eps, double one_minus_beta1,
                   double one_minus_beta2, double bias_corr1, double bias_corr2, void* stream);
/* numerics.py:31-42: op 0 out = a + b, op 1 out = a * s, op 2 out = max(a, 0) (NaN kept). */
int32_t dippm_elementwise_f64(int32_t op, const double* a, const double* b, double s, double* out, int64_t n,
                              void* stream);
/* numerics.py:23-28: c[M,N] = a[M,K] @ b[K,N], fp64 row-major. */
int32_t dippm_dgemm(const double* a, const double* b, double* c, int64_t M, int64_t K, int64_t N, void* stream);

/* ---------------------------------------------------------------------------
 * MIG-pick parity of the bf16 predict path (mig.py:32-45): graphs whose
 * bf16-predicted memory (y_pred [G,3] fp64, column 1) lies within band_mb of a profile
 * ceiling are re-scored in fp32.  Edges must be grouped by graph (edge_ptr [G+1]).
 *
 * Select (one launch): sel_idx [G] gets the band graphs in order, sel_node_ptr [G+1] int32 /
 * sel_edge_ptr [G+1] int64 the exclusive prefix sums of their node / edge counts (the
 * sub-batch's graph_ptr / edge_ptr), totals[3] = {count, nodes, edges} (device). */
int32_t dippm_mig_band_select(const double* y_pred, int64_t num_graphs, double band_mb, const int32_t* graph_ptr,
                              const int64_t* edge_ptr, int32_t* sel_idx, int32_t* sel_node_ptr, int64_t* sel_edge_ptr,
                              int64_t* totals, void* stream);
/* Gather the count selected graphs into a compact sub-batch: x_out [nodes, 32] f32, edges
 * re-based onto the sub-batch's node ids, fs_out [count, 5] fp64.  One CTA per graph. */
int32_t dippm_gather_graphs(const int32_t* sel_idx, int64_t count, const int32_t* sel_node_ptr,
                            const int64_t* sel_edge_ptr, const int32_t* graph_ptr, const int64_t* edge_ptr,
                            const float* x, const int64_t* src, const int64_t* dst, const double* fs, float* x_out,
                            int64_t* src_out, int64_t* dst_out, double* fs_out, void* stream);
/* y_pred[sel_idx[k]] = y_sub[k], mig[sel_idx[k]] = mig_sub[k] for k < count. */
int32_t dippm_scatter_rescore(const int32_t* sel_idx, int64_t count, const double* y_sub, const int8_t* mig_sub,
                              double* y_pred, int8_t* mig, void* stream);

/* ---------------------------------------------------------------------------
 * Native training-step executor: one batched bf16 training step (the BatchTrainer step of
 * trainer.py for a single rank: K1 CSR, forward with the fused readout, the fused head with
 * Huber loss and head backward, readout backward, the SAGE backward with the weight
 * gradients on a side stream, Adam + operand repack) issued from C++ in ONE call, so the
 * host cost of a step is its ~18 kernel launches instead of ~18 Python-level library calls
 * (gnn.py:383-405 objective, numerics.py:93-114 Adam -- the same kernels, arguments and
 * order as the Python orchestration in device.py, which the GPU tests compare bit for bit).
 *
 * The plan holds every device pointer that stays fixed across steps (model, workspace and
 * CSR buffers sized for the workspace capacity); dippm_train_plan_init creates the side
 * stream and the fork/join events, dippm_train_plan_destroy releases them. */
typedef struct dippm_train_plan {
  /* model: flat fp64 masters / Adam moments, fp32 gradients and compute copy (device.Layout) */
  int32_t hp, u_width;
  double *params, *m, *v;
  float *grads, *p32;
  int64_t n_params;
  int64_t* t_dev;             /* device Adam step counter */
  const double* norm;         /* double[16] */
  dippm_act_t Wf[3], Wd[3];   /* forward / dgrad operand copies (Wd[0] unused) */
  dippm_act_t W1h, W2h;
  const dippm_pack_seg_t* segs;
  int32_t n_segs;
  int64_t off_w[3], off_b[3]; /* sage{l}.w_self / sage{l}.bias offsets in the flat layout */
  int64_t off_fc1w, off_fc1b, off_fc2w, off_fc2b, off_fc3w, off_fc3b;
  /* workspace (capacity ws_N nodes, ws_G graphs, ws_E edges) */
  int64_t ws_N, ws_G, ws_E;
  dippm_act_t A[3], B[3];
  uint32_t* relu_bits;        /* [3][hp/32][ws_N] */
  float *pool_part, *pool_graph;
  dippm_act_t u, x2, x3, d2, d1;
  float* dhead_f32;           /* [2][ws_G][hp] */
  uint32_t* head_bits;        /* [hp/32][ws_G] */
  float *out, *dout, *du;
  double *loss, *row_loss;
  int32_t* head_sync;
  float* colsum;              /* layer 2's deferred bias partials ... */
  float* colsum3;             /* ... and layer 3's (folded by their weight-gradient GEMMs) */
  int32_t* colsum_sync;
  float* splitk;
  int32_t* tile_sync;
  /* K1 CSR outputs and scratch (capacity) */
  int32_t *rowptr, *col, *deg, *t_rowptr, *t_col, *bad, *node_graph;
  float* inv_deg;
  void* csr_ws;
  size_t csr_ws_bytes;
  /* hyper-parameters */
  double dropout_p, keep_scale, delta, grad_den, lr, beta1, beta2, eps;
  uint64_t seed;
  /* created by dippm_train_plan_init */
  void* side_stream;
  void* ev[4];                /* fork events (layers 3, 2, 1) and the join */
  void* graph_exec;           /* dippm_train_step_graphed's executable graph (NULL until first use) */
  void* capture_stream;       /* the stream dippm_train_step_graphed records on (never the legacy stream) */
  void* head_done;            /* recorded by each step after its fused head launch (also inside a
                                 captured step); dippm_train_prep waits on the latest record, so the
                                 next batch's K1 runs beside this step's backward */
} dippm_train_plan_t;

/* One batch's K1 outputs: the CSR / transposed CSR, the node->graph map and the layer-1
 * operand A1 = [x | agg x | 0] (bf16, [N, 128] view).  dippm_train_prep builds a set ahead of
 * the step, on another stream, so K1 runs beside the previous step instead of at the head of
 * this one (its CTAs fill the SMs the previous step's kernel tails and the fused head leave
 * idle); the plan's own CSR buffers + A[0] form the default set. */
typedef struct dippm_csr_set {
  int32_t *rowptr, *col, *deg, *t_rowptr, *t_col, *node_graph;
  float* inv_deg;
  void* csr_ws;
  size_t csr_ws_bytes;
  dippm_act_t a1;
  int64_t cap_N, cap_E;       /* capacity (nodes, edges) */
} dippm_csr_set_t;

typedef struct dippm_train_batch {
  const float* x;             /* [N, 32] */
  const int64_t *src, *dst;   /* [E] batch-global node ids */
  const int32_t* graph_ptr;   /* [G+1] */
  const int64_t* edge_ptr;    /* [G+1] edges grouped by graph, or NULL (global CSR path) */
  const double *fs, *y;       /* [G, 5], [G, 3] */
  int64_t N, E, G;
  int32_t max_nodes, max_edges; /* largest graph (grouped CSR path) */
  double* loss_out;           /* double[4] for this step's loss, or NULL: plan->loss */
  int32_t* bad_out;           /* int32[1] for this step's CSR edge flag, or NULL: plan->bad */
  const dippm_csr_set_t* csr; /* K1 outputs already built by dippm_train_prep (the step's stream
                                 must be ordered after that prep), or NULL: the step runs K1
                                 itself into the plan's buffers */
  int32_t no_adam;            /* 1: stop once every gradient is final (data parallel: the caller
                                 all-reduces plan->grads, then runs dippm_adam_pack; the head has
                                 already advanced plan->t_dev) */
} dippm_train_batch_t;

int32_t dippm_train_plan_init(dippm_train_plan_t* plan);
int32_t dippm_train_plan_destroy(dippm_train_plan_t* plan);
/* One step; the loss (double[4], as dippm_huber) goes to batch->loss_out (else plan->loss),
 * the CSR edge flag to batch->bad_out (else plan->bad): per-step slots let the caller read
 * them back on another stream while the next step runs.  Returns DIPPM_ERR_ARG (nothing launched) for a batch the plan cannot run
 * (larger than its capacity, or a head batch outside the fused head's range). */
int32_t dippm_train_step(const dippm_train_plan_t* plan, const dippm_train_batch_t* batch, void* stream);
/* The same step as ONE CUDA-graph launch: the step is captured (recorded, not run), the
 * plan's executable graph is updated in place with the new kernel arguments (ragged N / E
 * change grids and arguments, not the topology; a topology change re-instantiates) and
 * launched on `stream` -- no per-kernel launch gaps on the device. */
int32_t dippm_train_step_graphed(dippm_train_plan_t* plan, const dippm_train_batch_t* batch, void* stream);
/* K1 of `batch` into `set` on `stream` (grouped per-graph CSR + A1 in one launch, or the
 * global CSR path + the layer-1 aggregation), ordered after the fused head of the step last
 * launched with this plan (plan->head_done: K1's CTAs then share the SMs with that step's
 * backward instead of its GEMM mainloops); the edge flag goes to batch->bad_out (else
 * plan->bad).  batch->csr is ignored.  A later dippm_train_step with batch->csr = set, on a
 * stream ordered after this one, skips K1.  The caller keeps `set` untouched until that step
 * has finished (the next prep into it must be ordered after the step). */
int32_t dippm_train_prep(const dippm_train_plan_t* plan, const dippm_train_batch_t* batch, const dippm_csr_set_t* set,
                         void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DIPPM_B200_H_ */
