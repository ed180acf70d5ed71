// Native training-step executor (include/dippm_b200.h, dippm_train_step): the batched bf16
// training step of trainer.py / device.py for one rank, issued from C++ in one call.
//
// The reference step (gnn.py:383-405 objective, numerics.py:93-114 Adam) runs as the same
// kernels with the same arguments and in the same order as the Python orchestration
// (device.Engine.forward / loss / backward / adam_step with the fused head and the
// side-stream weight gradients); tests/test_gpu_step_native.py checks the two give
// bit-identical parameters.  Only the launch sequence moves here: the host cost of a step
// drops from ~18 Python-level library calls (~0.8 ms, more than the 0.73 ms the GPU needs,
// so the end-to-end path was host-bound) to the kernel launches themselves.
#include <cuda_runtime.h>

#include <cstdlib>

#include "common.cuh"

namespace {

using namespace dippm;

dippm_act_t at_col(dippm_act_t a, int64_t c) {  // view starting at column c (ActBuf.view(c))
  const int64_t elem = a.dtype == DIPPM_DT_BF16 ? 2 : 4;
  a.data = static_cast<char*>(a.data) + c * elem;
  return a;
}
constexpr dippm_act_t kNullAct{nullptr, 0, 0, 0};
dippm_act_t f32_act(const void* p, int64_t ld) { return dippm_act_t{const_cast<void*>(p), ld, 0, DIPPM_DT_F32}; }

dippm_gemm_args_t gemm_defaults() {
  dippm_gemm_args_t a{};
  a.splits = 1;
  a.gate_scale = 1.0;
  a.out_scale = 1.0;
  return a;
}

constexpr int64_t kGroupedMaxGraphs = 8192;  // device.GROUPED_MAX_GRAPHS / GROUPED_MAX_EDGES
constexpr int64_t kGroupedMaxEdges = 8192;

#define STEP_CALL(expr)                \
  do {                                 \
    const int32_t _rc = (expr);        \
    if (_rc != DIPPM_OK) return _rc;   \
  } while (0)

// the plan's own K1 buffers (+ A[0]) as a set: the default when the batch brings none
dippm_csr_set_t plan_set(const dippm_train_plan_t* P) {
  dippm_csr_set_t c{};
  c.rowptr = P->rowptr;
  c.col = P->col;
  c.deg = P->deg;
  c.t_rowptr = P->t_rowptr;
  c.t_col = P->t_col;
  c.node_graph = P->node_graph;
  c.inv_deg = P->inv_deg;
  c.csr_ws = P->csr_ws;
  c.csr_ws_bytes = P->csr_ws_bytes;
  c.a1 = P->A[0];
  c.cap_N = P->ws_N;
  c.cap_E = P->ws_E;
  return c;
}

// ---- K1: CSR + transposed CSR (device.build_batch_csr) and the layer-1 operand
// A1 = [x | agg x] (Engine.forward's first aggregation)
int32_t build_k1(const dippm_train_batch_t* b, const dippm_csr_set_t& c, int32_t* bad, cudaStream_t s) {
  const int64_t N = b->N, G = b->G;
  DIPPM_ARG_CHECK(N <= c.cap_N && b->E <= c.cap_E && c.a1.data && c.a1.dtype == DIPPM_DT_BF16,
                  "train_step: CSR set (capacity %lld nodes, %lld edges) for %lld nodes, %lld edges",
                  (long long)c.cap_N, (long long)c.cap_E, (long long)N, (long long)b->E);
  const bool grouped = b->edge_ptr && G <= kGroupedMaxGraphs && b->max_edges <= kGroupedMaxEdges &&
                       b->max_nodes <= kGroupedMaxEdges;
  if (grouped) {
    DIPPM_ARG_CHECK(c.csr_ws_bytes >= dippm_csr_grouped_workspace_bytes(G, b->E), "train_step: CSR workspace");
    // + the layer-1 operand [x | agg x] while each graph's CSR is in shared memory
    return dippm_build_csr_grouped_l1(b->src, b->dst, b->graph_ptr, b->edge_ptr, G, N, b->E, b->max_nodes,
                                      b->max_edges, c.rowptr, c.col, c.deg, c.inv_deg, c.t_rowptr, c.t_col, bad,
                                      c.node_graph, c.csr_ws, c.csr_ws_bytes, b->x, c.a1, s);
  }
  DIPPM_ARG_CHECK(c.csr_ws_bytes >= dippm_csr_workspace_bytes(N, b->E), "train_step: CSR workspace");
  STEP_CALL(dippm_node_graph(b->graph_ptr, G, c.node_graph, s));
  STEP_CALL(dippm_build_csr(b->src, b->dst, b->E, N, c.rowptr, c.col, c.deg, c.inv_deg, c.t_rowptr, c.t_col, bad,
                            c.csr_ws, c.csr_ws_bytes, s));
  return dippm_sage_aggregate(f32_act(b->x, 32), at_col(c.a1, 32), c.a1, N, 32, c.rowptr, c.col, c.inv_deg, s);
}

}  // namespace

extern "C" {

int32_t dippm_train_plan_init(dippm_train_plan_t* plan) {
  DIPPM_ARG_CHECK(plan, "train_plan_init: NULL plan");
  cudaStream_t s = nullptr;
  DIPPM_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  plan->side_stream = s;
  DIPPM_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  plan->capture_stream = s;
  cudaEvent_t hd = nullptr;
  DIPPM_CUDA_CHECK(cudaEventCreateWithFlags(&hd, cudaEventDisableTiming));
  plan->head_done = hd;
  for (int i = 0; i < 4; ++i) {
    cudaEvent_t e = nullptr;
    DIPPM_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    plan->ev[i] = e;
  }
  return DIPPM_OK;
}

int32_t dippm_train_plan_destroy(dippm_train_plan_t* plan) {
  if (!plan) return DIPPM_OK;
  if (plan->graph_exec) {
    cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(plan->graph_exec));
    plan->graph_exec = nullptr;
  }
  for (int i = 0; i < 4; ++i)
    if (plan->ev[i]) {
      cudaEventDestroy(static_cast<cudaEvent_t>(plan->ev[i]));
      plan->ev[i] = nullptr;
    }
  if (plan->head_done) {
    cudaEventDestroy(static_cast<cudaEvent_t>(plan->head_done));
    plan->head_done = nullptr;
  }
  for (void** st : {&plan->side_stream, &plan->capture_stream})
    if (*st) {
      cudaStreamDestroy(static_cast<cudaStream_t>(*st));
      *st = nullptr;
    }
  return DIPPM_OK;
}

int32_t dippm_train_step(const dippm_train_plan_t* P, const dippm_train_batch_t* b, void* stream) {
  DIPPM_ARG_CHECK(P && b && P->side_stream, "train_step: plan not initialised");
  DIPPM_ARG_CHECK(b->N >= 1 && b->G >= 1 && b->E >= 0, "train_step: empty batch");
  DIPPM_ARG_CHECK(b->N <= P->ws_N && b->G <= P->ws_G && (b->csr || b->E <= P->ws_E),
                  "train_step: batch (%lld nodes, %lld graphs, %lld edges) exceeds the plan's capacity",
                  (long long)b->N, (long long)b->G, (long long)b->E);
  DIPPM_ARG_CHECK(b->G <= dippm_head_fused_max_graphs() && P->hp <= 512 && P->u_width <= 576 &&
                      P->A[0].dtype == DIPPM_DT_BF16,
                  "train_step: batch outside the fused bf16 head's range");
  DIPPM_ARG_CHECK(!b->csr || (b->N <= b->csr->cap_N && b->E <= b->csr->cap_E),
                  "train_step: batch larger than its prepared CSR set");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaStream_t side = static_cast<cudaStream_t>(P->side_stream);
  const int64_t N = b->N, G = b->G, hp = P->hp;
  const int32_t d_in[3] = {32, (int32_t)hp, (int32_t)hp};
  const int64_t bits_words = (hp / 32) * P->ws_N;
  double* loss_out = b->loss_out ? b->loss_out : P->loss;
  int32_t* bad = b->bad_out ? b->bad_out : P->bad;
  auto bits = [&](int i) { return P->relu_bits + i * bits_words; };
  auto p32 = [&](int64_t off) { return P->p32 + off; };
  auto g32 = [&](int64_t off) { return P->grads + off; };

  // ---- K1 (here, or already run by dippm_train_prep into the batch's set)
  const dippm_csr_set_t C = b->csr ? *b->csr : plan_set(P);
  if (!b->csr) STEP_CALL(build_k1(b, C, bad, s));

  // ---- forward (Engine.forward, train mode, head deferred to the backward)
  for (int i = 0; i < 3; ++i) {
    if (i > 0)
      STEP_CALL(dippm_sage_aggregate(P->A[i], at_col(P->A[i], hp), kNullAct, N, (int32_t)hp, C.rowptr, C.col,
                                     C.inv_deg, s));
    dippm_gemm_args_t a = gemm_defaults();
    a.kind = DIPPM_GEMM_FWD;
    a.M = N;
    a.N = hp;
    a.K = 2 * d_in[i];
    a.a = i == 0 ? C.a1 : P->A[i];
    a.b = P->Wf[i];
    a.b_mn_major = 1;
    a.bias = p32(P->off_b[i]);
    a.relu = 1;
    a.out = i < 2 ? P->A[i + 1] : kNullAct;  // h3 itself is never stored (its readout and mask are)
    a.relu_bits = bits(i);
    a.bits_ld = i == 2 ? 0 : P->ws_N;          // h3's mask row-major: read per row by the readout backward
    if (i == 2) {
      a.pool_partial = P->pool_part;
      a.pool_graph = P->pool_graph;
      a.node_graph = C.node_graph;
      a.graph_ptr = b->graph_ptr;
    }
    STEP_CALL(dippm_gemm(&a, 0, s));
  }
  STEP_CALL(dippm_pool_combine(P->pool_part, P->pool_graph, b->graph_ptr, G, (int32_t)hp, b->fs, P->norm, P->u, s));

  // ---- fused head: forward + Huber loss + head backward (+ the Adam step counter)
  const int drop = P->dropout_p > 0.0 ? 2 : 0;
  dippm_head_args_t h{};
  h.G = G;
  h.hp = (int32_t)hp;
  h.u_width = P->u_width;
  h.u = P->u.data;
  h.w1 = P->W1h.data;
  h.w2 = P->W2h.data;
  h.b1 = p32(P->off_fc1b);
  h.b2 = p32(P->off_fc2b);
  h.w3 = p32(P->off_fc3w);
  h.b3 = p32(P->off_fc3b);
  h.x2 = P->x2.data;
  h.x3 = P->x3.data;
  h.bits = P->head_bits;
  h.bits_ld = P->ws_G;
  h.drop_mode = drop;
  h.drop_p = P->dropout_p;
  h.keep_scale = (float)P->keep_scale;
  h.seed1 = P->seed * 2;
  h.seed2 = P->seed * 2 + 1;
  h.seed_dev = drop == 2 ? P->t_dev : nullptr;
  h.out = P->out;
  h.norm = P->norm;
  h.y_raw = b->y;
  h.delta = P->delta;
  h.grad_den = P->grad_den;
  h.loss_out = loss_out;
  h.row_loss = P->row_loss;
  h.dout = P->dout;
  h.d2 = P->d2.data;
  h.d1 = P->d1.data;
  h.d2f = P->dhead_f32;
  h.d1f = P->dhead_f32 + P->ws_G * hp;
  h.gw1 = g32(P->off_fc1w);
  h.gb1 = g32(P->off_fc1b);
  h.gw2 = g32(P->off_fc2w);
  h.gb2 = g32(P->off_fc2b);
  h.gw3 = g32(P->off_fc3w);
  h.gb3 = g32(P->off_fc3b);
  h.du = P->du;
  h.train = 1;
  h.step_counter = P->t_dev;  // this step's t += 1 (no separate dippm_step_counter launch)
  h.sync = P->head_sync;
  // dW1 / dW2: weight-gradient GEMMs on the side stream (below); DIPPM_HEAD_WGRAD_INLINE=1
  // keeps them in the head kernel (A/B switch, as device.HEAD_WGRAD_DEFER)
  static const bool head_wgrad_inline = getenv("DIPPM_HEAD_WGRAD_INLINE") && getenv("DIPPM_HEAD_WGRAD_INLINE")[0] == '1';
  if (!head_wgrad_inline) {
    h.gw1 = h.gw2 = nullptr;
    h.defer_reduce = 1;  // column sums + loss: dippm_head_reduce on the side stream
  }
  STEP_CALL(dippm_head_fused(&h, s));
  if (P->head_done) {  // the next batch's K1 (dippm_train_prep) may start from here
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    DIPPM_CUDA_CHECK(cudaStreamIsCapturing(s, &cs));
    DIPPM_CUDA_CHECK(cudaEventRecordWithFlags(static_cast<cudaEvent_t>(P->head_done), s,
                                              cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal
                                                                                  : cudaEventRecordDefault));
  }

  // ---- weight gradients (side stream): one [width, hp] = A^T dz GEMM, split over K in fixed order
  auto wgrad = [&](const dippm_act_t& A, const dippm_act_t& dz, int64_t width, int64_t rows, int64_t off_out,
                   float* bias_partial, float* bias_grad) -> int32_t {
    dippm_gemm_args_t w = gemm_defaults();
    w.kind = DIPPM_GEMM_WGRAD;
    w.M = width;
    w.N = hp;
    w.K = rows;
    w.a = A;
    w.a_mn_major = 1;
    w.b = dz;
    w.b_mn_major = 1;
    w.out = f32_act(g32(off_out), hp);
    w.c = P->splitk;
    w.ldc = hp;
    w.splits = dippm_wgrad_splits(width, hp, rows);
    w.tile_sync = P->tile_sync;
    w.bias_partial = bias_partial;
    w.bias_grad = bias_grad;
    return dippm_gemm(&w, 0, side);
  };
  // the head's dW2 = x2^T d2 and dW1 = u^T d1 (device.Engine.backward, head_wgrads)
  if (!head_wgrad_inline) {
    cudaEvent_t ev = static_cast<cudaEvent_t>(P->ev[3]);
    DIPPM_CUDA_CHECK(cudaEventRecord(ev, s));
    DIPPM_CUDA_CHECK(cudaStreamWaitEvent(side, ev, 0));
    STEP_CALL(dippm_head_reduce(&h, side));
    STEP_CALL(wgrad(P->x2, P->d2, hp, G, P->off_fc2w, nullptr, nullptr));
    STEP_CALL(wgrad(P->u, P->d1, P->u_width, G, P->off_fc1w, nullptr, nullptr));
  }

  // Adam split at sage3's first parameter (flat layout sage1 | sage2 | sage3 | fc1..fc3,
  // gnn.py:488-491): the upper range's operand-copy segments, rebased; DIPPM_SPLIT_ADAM=0 keeps
  // one launch at the end (A/B switch).  Element-wise update: the same results either way.
  static const bool split_env = !(getenv("DIPPM_SPLIT_ADAM") && getenv("DIPPM_SPLIT_ADAM")[0] == '0');
  const int64_t off3 = P->off_w[2];
  dippm_pack_seg_t seg_lo[DIPPM_MAX_PACK_SEGS], seg_hi[DIPPM_MAX_PACK_SEGS];
  int n_lo = 0, n_hi = 0;
  bool split_adam = split_env && !b->no_adam && off3 % 8 == 0 && P->n_segs <= DIPPM_MAX_PACK_SEGS;
  for (int k = 0; split_adam && k < P->n_segs; ++k) {
    dippm_pack_seg_t sg = P->segs[k];
    if (sg.src_off >= off3) {
      sg.src_off -= off3;
      seg_hi[n_hi++] = sg;
    } else if (sg.src_off + sg.rows * sg.cols <= off3) {
      seg_lo[n_lo++] = sg;
    } else {
      split_adam = false;  // a segment straddles the split: one launch
    }
  }

  // ---- SAGE backward: dgrad chain on the main stream, weight gradients on the side stream
  for (int i = 2; i >= 0; --i) {
    const dippm_act_t Bi = P->B[i];
    // layers 2-3: the bias partial rows are folded by the layer's weight-gradient GEMM (deferred mode)
    float* part = i == 2 ? P->colsum3 : P->colsum;
    if (i == 2) {
      STEP_CALL(dippm_readout_aggregate_t(P->du, hp, b->graph_ptr, C.node_graph, kNullAct, Bi, (int32_t)hp, N,
                                          C.t_rowptr, C.t_col, C.inv_deg, part, nullptr, P->colsum_sync, bits(2),
                                          0, s));
    } else if (i == 1) {
      STEP_CALL(dippm_sage_aggregate_t(Bi, (int32_t)hp, N, 1, C.t_rowptr, C.t_col, C.inv_deg, part, nullptr,
                                       P->colsum_sync, s));
    }
    // weight gradient [2d (+1: layer 1's ones column = the bias row), hp] on the side stream
    cudaEvent_t ev = static_cast<cudaEvent_t>(P->ev[2 - i]);
    DIPPM_CUDA_CHECK(cudaEventRecord(ev, s));
    DIPPM_CUDA_CHECK(cudaStreamWaitEvent(side, ev, 0));
    const int64_t width = 2 * d_in[i] + (i == 0 ? 1 : 0);
    STEP_CALL(wgrad(i == 0 ? C.a1 : P->A[i], Bi, width, N, P->off_w[i], i > 0 ? part : nullptr,
                    i > 0 ? g32(P->off_b[i]) : nullptr));
    if (i == 0) break;
    dippm_gemm_args_t g = gemm_defaults();
    g.kind = DIPPM_GEMM_GATE;
    g.M = N;
    g.N = d_in[i];
    g.K = 2 * hp;
    g.a = Bi;
    g.b = P->Wd[i];
    g.out = P->B[i - 1];
    g.gate = P->A[i];
    g.gate_bits = bits(i - 1);
    g.bits_ld = P->ws_N;
    STEP_CALL(dippm_gemm(&g, 0, s));
    if (i == 2 && split_adam) {
      // sage3 + head gradients are final (head reductions / WGRADs and WGRAD_3 ran on the side
      // stream); once GATE_3, the last reader of sage3's dgrad copy, is done, their Adam update
      // runs on the side stream beside agg^T_2 -- off the step's tail
      cudaEvent_t ev = static_cast<cudaEvent_t>(P->ev[3]);
      DIPPM_CUDA_CHECK(cudaEventRecord(ev, s));
      DIPPM_CUDA_CHECK(cudaStreamWaitEvent(side, ev, 0));
      STEP_CALL(dippm_adam_pack(P->params + off3, P->m + off3, P->v + off3, P->grads + off3, 1.0,
                                P->n_params - off3, 0, P->t_dev, P->lr, P->beta1, P->beta2, P->eps, 1, P->p32 + off3,
                                seg_hi, n_hi, side));
    }
  }
  cudaEvent_t join = static_cast<cudaEvent_t>(P->ev[3]);
  DIPPM_CUDA_CHECK(cudaEventRecord(join, side));
  DIPPM_CUDA_CHECK(cudaStreamWaitEvent(s, join, 0));

  if (b->no_adam) return DIPPM_OK;  // data parallel: the caller all-reduces, then runs Adam
  // ---- Adam (t already advanced by the head) + refresh of every operand copy: sage1 + sage2
  // here (sage3 + head already updated on the side stream), or everything
  if (split_adam)
    STEP_CALL(dippm_adam_pack(P->params, P->m, P->v, P->grads, 1.0, off3, 0, P->t_dev, P->lr, P->beta1, P->beta2,
                              P->eps, 1, P->p32, seg_lo, n_lo, s));
  else
    STEP_CALL(dippm_adam_pack(P->params, P->m, P->v, P->grads, 1.0, P->n_params, 0, P->t_dev, P->lr, P->beta1,
                              P->beta2, P->eps, 1, P->p32, P->segs, P->n_segs, s));
  return DIPPM_OK;
}

int32_t dippm_train_prep(const dippm_train_plan_t* P, const dippm_train_batch_t* b, const dippm_csr_set_t* set,
                         void* stream) {
  DIPPM_ARG_CHECK(P && b && set, "train_prep: NULL argument");
  DIPPM_ARG_CHECK(b->N >= 1 && b->G >= 1 && b->E >= 0, "train_prep: empty batch");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (P->head_done) DIPPM_CUDA_CHECK(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(P->head_done), 0));
  return build_k1(b, *set, b->bad_out ? b->bad_out : P->bad, s);
}

int32_t dippm_train_step_graphed(dippm_train_plan_t* P, const dippm_train_batch_t* b, void* stream) {
  DIPPM_ARG_CHECK(P, "train_step_graphed: NULL plan");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaStream_t cap = static_cast<cudaStream_t>(P->capture_stream);
  DIPPM_ARG_CHECK(cap, "train_step_graphed: plan not initialised");
  // record on the plan's own stream (capture cannot start on the legacy default stream); the
  // recorded graph is launched on `stream`, so it runs in that stream's order
  DIPPM_CUDA_CHECK(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
  const int32_t rc = dippm_train_step(P, b, cap);
  cudaGraph_t g = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(cap, &g);
  if (rc != DIPPM_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  DIPPM_CUDA_CHECK(ce);
  cudaGraphExec_t ex = static_cast<cudaGraphExec_t>(P->graph_exec);
  bool updated = false;
  if (ex) {
    cudaGraphExecUpdateResultInfo info{};
    updated = cudaGraphExecUpdate(ex, g, &info) == cudaSuccess;
    if (!updated) {
      cudaGetLastError();  // clear the update failure: re-instantiate below
      cudaGraphExecDestroy(ex);
      P->graph_exec = ex = nullptr;
    }
  }
  if (!updated) {
    const cudaError_t ie = cudaGraphInstantiate(&ex, g, 0);
    if (ie != cudaSuccess) {
      cudaGraphDestroy(g);
      return cuda_status(ie, "train_step_graphed: instantiate");
    }
    P->graph_exec = ex;
  }
  cudaGraphDestroy(g);
  DIPPM_CUDA_CHECK(cudaGraphLaunch(ex, s));
  return DIPPM_OK;
}

}  // extern "C"
