"""Batched training step — the public throughput API for DIPPM training on B200.

`BatchTrainer.step_host(...)` is the end-to-end call a user makes with a
collated batch in host memory: H2D of the batch, K1 CSR build, train-mode
forward (device dropout masks), Huber loss, full backward, optional
data-parallel gradient all-reduce, fused Adam + repack, and a D2H read of the
loss.  `step_resident(batch)` is the same step for a batch already in HBM.

The objective per step is the reference's batch objective (gnn.py:383-405:
mean over the batch of the per-graph Huber loss) with train-mode dropout;
Adam follows numerics.py:93-114 on fp64 masters.
"""

from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np
import torch

from . import _lib
from . import device as dev
from .device import Batch, Engine, Workspace, build_batch_csr
from .errors import NonFinite, ShapeMismatch

# DIPPM_NATIVE_STEP=0 keeps the Python-orchestrated step (A/B switch; same kernels and order)
NATIVE_STEP = os.environ.get("DIPPM_NATIVE_STEP", "1") != "0"
# DIPPM_NATIVE_GRAPHED=0: submit() launches the native step's kernels one by one instead of as
# one updated CUDA graph
NATIVE_GRAPHED = os.environ.get("DIPPM_NATIVE_GRAPHED", "1") != "0"
# DIPPM_NATIVE_PREP=0: the native step runs K1 (CSR build + layer-1 operand) at its head instead
# of ahead of it on a separate stream (dippm_train_prep), where it overlaps the previous step
NATIVE_PREP = os.environ.get("DIPPM_NATIVE_PREP", "1") != "0"


class CsrBuffers:
    """One batch's K1 outputs for the native step (dippm_csr_set_t): CSR and transposed CSR,
    node -> graph map, and the layer-1 operand A1 = [x | agg x | 1 | 0] (bf16 [N, 128], the
    constant ones column as in Workspace).  Built by dippm_train_prep on a side stream ahead of
    the step that reads it; `free` marks the last step that read it, `ready` the prep."""

    def __init__(self, N: int, E: int, G: int, device):
        lib = _lib.load()
        i32 = dict(dtype=torch.int32, device=device)
        N, E, G = max(1, int(N)), max(1, int(E)), max(1, int(G))
        self.N, self.E, self.G = N, E, G
        self.rowptr, self.t_rowptr = torch.empty(N + 1, **i32), torch.empty(N + 1, **i32)
        self.col, self.t_col = torch.empty(E, **i32), torch.empty(E, **i32)
        self.deg, self.node_graph = torch.empty(N, **i32), torch.empty(N, **i32)
        self.inv_deg = torch.empty(N, dtype=torch.float32, device=device)
        nbytes = max(lib.dippm_csr_grouped_workspace_bytes(G, E), lib.dippm_csr_workspace_bytes(N, E))
        self.csr_ws = torch.empty(nbytes, dtype=torch.uint8, device=device)
        self.a1 = dev.ActBuf(N, 4 * dev.FEATURE_WIDTH, dev.DT_BF16, device)
        self.a1.t[:, 2 * dev.FEATURE_WIDTH:].zero_()
        self.a1.t[:, 2 * dev.FEATURE_WIDTH] = 1.0
        p = dev._p
        self.s = _lib.CsrSet(p(self.rowptr), p(self.col), p(self.deg), p(self.t_rowptr), p(self.t_col),
                             p(self.node_graph), p(self.inv_deg), p(self.csr_ws), nbytes, self.a1.view(), N, E)
        self.free, self.ready = None, torch.cuda.Event()

    def fits(self, b: Batch) -> bool:
        return b.N <= self.N and b.E <= self.E and b.G <= self.G


class NativeStep:
    """dippm_train_step's plan for one (engine, workspace): every fixed device pointer of the
    bf16 single-rank training step, plus capacity-sized K1 CSR buffers.  One library call per
    step replaces the ~18 Python-level launches of Engine.forward / loss / backward / adam_step
    (the same kernels, arguments and order; tests/test_gpu_step_native.py compares them)."""

    def __init__(self, trainer: "BatchTrainer", max_edges: int):
        eng, ws = trainer.engine, trainer.ws
        L, hp = eng.L, eng.L.hp
        lib = _lib.load()
        self.ws, self.E = ws, max(1, int(max_edges))
        d = eng.device
        i32 = dict(dtype=torch.int32, device=d)
        N, G, E = ws.N, ws.G, self.E
        self.rowptr, self.t_rowptr = torch.empty(N + 1, **i32), torch.empty(N + 1, **i32)
        self.col, self.t_col = torch.empty(E, **i32), torch.empty(E, **i32)
        self.deg, self.node_graph = torch.empty(N, **i32), torch.empty(N, **i32)
        self.inv_deg = torch.empty(N, dtype=torch.float32, device=d)
        self.bad = torch.zeros(1, **i32)
        nbytes = max(lib.dippm_csr_grouped_workspace_bytes(G, E), lib.dippm_csr_workspace_bytes(N, E))
        self.csr_ws = torch.empty(nbytes, dtype=torch.uint8, device=d)
        p = self.plan = _lib.TrainPlan()
        ptr = dev._p
        p.hp, p.u_width = hp, L.u_width
        p.params, p.m, p.v, p.grads, p.p32 = ptr(eng.params), ptr(eng.m), ptr(eng.v), ptr(eng.grads), ptr(eng.p32)
        p.n_params, p.t_dev, p.norm = L.total, ptr(eng.t_dev), ptr(eng.norm)
        for i in range(3):
            p.Wf[i] = eng.Wf[i].view()
            p.Wd[i] = eng.Wd[i].view() if eng.Wd[i] is not None else dev.NULL_ACT
            p.off_w[i], p.off_b[i] = L.offsets[f"sage{i + 1}.w_self"], L.offsets[f"sage{i + 1}.bias"]
            p.A[i], p.B[i] = ws.A[i].view(0), ws.B[i].view(0)
        p.W1h, p.W2h = eng.W1h.view(), eng.W2h.view()
        p.segs, p.n_segs = C.cast(eng._segs, C.c_void_p), len(eng._segs)
        p.off_fc1w, p.off_fc1b = L.offsets["fc1.w"], L.offsets["fc1.b"]
        p.off_fc2w, p.off_fc2b = L.offsets["fc2.w"], L.offsets["fc2.b"]
        p.off_fc3w, p.off_fc3b = L.offsets["fc3.w"], L.offsets["fc3.b"]
        p.ws_N, p.ws_G, p.ws_E = N, G, E
        p.relu_bits, p.pool_part, p.pool_graph = ptr(ws.relu_bits), ptr(ws.pool_part), ptr(ws.pool_graph)
        p.u, p.x2, p.x3, p.d2, p.d1 = ws.u.view(), ws.x2.view(), ws.x3.view(), ws.d2.view(), ws.d1.view()
        p.dhead_f32, p.head_bits = ptr(ws.dhead_f32), ptr(ws.head_bits)
        p.out, p.dout, p.du, p.loss, p.row_loss = ptr(ws.out), ptr(ws.dout), ptr(ws.du), ptr(ws.loss), ptr(ws.row_loss)
        p.head_sync, p.colsum, p.colsum3, p.colsum_sync = (ptr(ws.head_sync), ptr(ws.colsum), ptr(ws.colsum3),
                                                            ptr(ws.colsum_sync))
        p.splitk, p.tile_sync = ptr(ws.splitk), ptr(ws.tile_sync)
        p.rowptr, p.col, p.deg, p.t_rowptr, p.t_col = (ptr(self.rowptr), ptr(self.col), ptr(self.deg),
                                                        ptr(self.t_rowptr), ptr(self.t_col))
        p.bad, p.node_graph, p.inv_deg = ptr(self.bad), ptr(self.node_graph), ptr(self.inv_deg)
        p.csr_ws, p.csr_ws_bytes = ptr(self.csr_ws), nbytes
        p.beta1, p.beta2, p.eps, p.grad_den = 0.9, 0.999, 1e-8, 0.0
        self.sync_hparams(trainer)
        _lib.check(lib.dippm_train_plan_init(C.byref(p)), "dippm_train_plan_init")
        self.batch = _lib.TrainBatch()
        self._fn, self._fn_graphed = lib.dippm_train_step, lib.dippm_train_step_graphed
        self._prep = lib.dippm_train_prep
        self._warm = False  # the plan's first step runs eagerly (kernel attributes, module loads)

    def sync_hparams(self, trainer: "BatchTrainer") -> None:
        """The trainer's current learning rate, Huber delta, dropout and seed (read every step,
        as the Python step reads them, so a schedule that changes trainer.lr takes effect)."""
        p = self.plan
        p.lr, p.delta, p.dropout_p = float(trainer.lr), float(trainer.delta), float(trainer.dropout_p)
        p.keep_scale = 1.0 / (1.0 - trainer.dropout_p) if trainer.dropout_p > 0 else 1.0
        p.seed = (trainer.seed * 131 + trainer.rank) & (2**64 - 1)

    def fits(self, b: Batch) -> bool:
        return b.N <= self.ws.N and b.G <= self.ws.G and b.E <= self.E

    def _fill(self, b: Batch, loss_out, bad_out, cset: CsrBuffers | None, no_adam: bool = False) -> _lib.TrainBatch:
        t = self.batch
        t.no_adam = 1 if no_adam else 0
        t.loss_out = loss_out
        t.bad_out = None if bad_out is None else bad_out.data_ptr()
        t.x, t.src, t.dst, t.graph_ptr = b.x.data_ptr(), b.src.data_ptr(), b.dst.data_ptr(), b.graph_ptr.data_ptr()
        t.edge_ptr = b.edge_ptr.data_ptr() if b.edge_ptr is not None else None
        t.fs, t.y = b.fs.data_ptr(), b.y.data_ptr()
        t.N, t.E, t.G, t.max_nodes, t.max_edges = b.N, b.E, b.G, b.max_nodes, b.max_edges
        t.csr = C.pointer(cset.s) if cset is not None else None
        return t

    def prep(self, b: Batch, cset: CsrBuffers, stream: torch.cuda.Stream,
             bad_out: torch.Tensor | None = None) -> None:
        """K1 of batch b into cset on `stream` (dippm_train_prep); the caller orders the step
        that reads cset after it."""
        t = self._fill(b, None, bad_out, None)
        _lib.check(self._prep(C.byref(self.plan), C.byref(t), C.byref(cset.s), stream.cuda_stream),
                   "dippm_train_prep")

    def step(self, b: Batch, loss_out: int | None = None, bad_out: torch.Tensor | None = None,
             graphed: bool = False, cset: CsrBuffers | None = None, no_adam: bool = False) -> None:
        """graphed: run the step as one CUDA-graph launch (dippm_train_step_graphed; the
        ragged host-batch path, where per-batch torch graphs cannot be reused).  cset: K1
        outputs already built by prep() (else the step runs K1 itself).  no_adam: stop at the
        final gradients (data parallel: the caller all-reduces them and runs Adam)."""
        t = self._fill(b, loss_out, bad_out, cset, no_adam)
        fn = self._fn_graphed if graphed and self._warm and not torch.cuda.is_current_stream_capturing() else self._fn
        _lib.check(fn(C.byref(self.plan), C.byref(t), torch.cuda.current_stream().cuda_stream), "dippm_train_step")
        self._warm = True
        b.bad = self.bad if bad_out is None else bad_out

    def __del__(self):
        try:
            _lib.load().dippm_train_plan_destroy(C.byref(self.plan))
        except Exception:
            pass


class BatchTrainer:
    def __init__(self, model, precision: str = "bf16", lr: float = 2.754e-5, seed: int = 0, dropout: bool = True,
                 huber_delta: float = 1.0, allreduce=None, world_size: int = 1, rank: int = 0, device=None,
                 use_graphs: bool = False):
        self.model = model
        self.engine = Engine(model.hidden, precision, device, arch=getattr(model, "arch", "sage"))
        self.engine.set_params(model.param_items(), model.normalizer)
        self.lr, self.seed, self.delta = lr, seed, huber_delta
        self.dropout_p = model.dropout_p if dropout else 0.0
        self.allreduce = allreduce
        self.world_size, self.rank = world_size, rank
        self.use_graphs = use_graphs
        self._graphs, self._keep, self._warm = {}, [], False
        self._pool = torch.cuda.graph_pool_handle() if use_graphs else None
        self.steps = 0
        self.replayed_launches = 0  # kernels launched by graph replays (not seen by dippm_launch_count)
        self.ws = None
        self._slots = []
        self._slot_next = 0
        self._copy_stream = torch.cuda.Stream() if torch.cuda.is_available() else None
        self._loss_ring = [torch.zeros(1, dtype=torch.float64).pin_memory() for _ in range(64)]
        self._flag_ring = [torch.zeros(1, dtype=torch.int32).pin_memory() for _ in range(64)]
        self._loss_next = 0
        self._native = None
        self._csr_ring, self._csr_next = [None, None], 0
        if torch.cuda.is_available():  # native steps: per-step loss / flag slots and their read-back stream
            self._prep_stream = torch.cuda.Stream(self.engine.device)
            self._d2h_stream = torch.cuda.Stream(self.engine.device)
            self._loss_dev = torch.zeros(len(self._loss_ring), 4, dtype=torch.float64, device=self.engine.device)
            self._bad_dev = torch.zeros(len(self._loss_ring), dtype=torch.int32, device=self.engine.device)

    def reserve(self, max_nodes: int, max_graphs: int, max_edges: int | None = None) -> None:
        """Preallocate the workspace (and host-batch staging) for batches up to this size."""
        self.ws = Workspace(self.engine, max_nodes, max_graphs, train=True)
        self._native = None   # the native plan points into the old workspace
        self._graphs.clear()  # captured steps point into the old workspace
        self._keep.clear()
        e = max_edges if max_edges is not None else 2 * max_nodes
        d = self.engine.device
        self._slots = [{  # two host-batch staging slots (double buffering for submit())
            "x": torch.empty(max_nodes, dev.FEATURE_WIDTH, dtype=torch.float32, device=d),
            "src": torch.empty(e, dtype=torch.int64, device=d), "dst": torch.empty(e, dtype=torch.int64, device=d),
            "gp": torch.empty(max_graphs + 1, dtype=torch.int32, device=d),
            "fs": torch.empty(max_graphs, dev.STATIC_WIDTH, dtype=torch.float64, device=d),
            "y": torch.empty(max_graphs, 3, dtype=torch.float64, device=d),
            "ep": torch.empty(max_graphs + 1, dtype=torch.int64, device=d),
            "free": torch.cuda.Event(), "ready": torch.cuda.Event(),
        } for _ in range(2)]
        self._slot_next = 0

    def _ensure(self, b: Batch) -> None:
        if self.ws is None or b.N > self.ws.N or b.G > self.ws.G:
            self.reserve(max(b.N, 1), b.G)

    def step_resident(self, b: Batch, global_graphs: int | None = None) -> None:
        """One training step on a device-resident batch (no host synchronisation).

        Data parallel: the gradient denominator is the global batch
        (`global_graphs`, default G x world), so the all-reduced SUM of the
        per-rank gradients is the global batch mean (gnn.py:402-404).

        Native steps build the batch's CSR (K1) on a separate stream ahead of the step, ordered
        after the batch's uploads as they stood at its first step: a resident batch's tensors
        are not rewritten afterwards (upload a new Batch instead)."""
        self._ensure(b)
        self.steps += 1
        self.engine._uploaded = None  # the step moves the device parameters
        cset = self._resident_prep(b)
        if not self.use_graphs:
            self._step(b, global_graphs, cset=cset)
            self._release(cset)
            return
        # CUDA graphs: the trainer's first step runs eagerly (module load, kernel
        # attributes); afterwards each resident batch's step is captured once
        # and replayed.  Step-dependent values (Adam's t, the dropout stream)
        # live on the device, so replays advance them.
        hit = self._graphs.get(id(b))
        if hit is None:
            if not self._warm:
                self._step(b, global_graphs, cset=cset)
                self._release(cset)
                self._warm = True
                return
            hit = self.capture(b, global_graphs, cset)
        hit[0].replay()
        self._release(cset)
        self.replayed_launches += hit[1]  # (the prep's K1 launch is counted by the library)

    def capture(self, b: Batch, global_graphs: int | None = None, cset: CsrBuffers | None = None):
        """Record (without executing) the training step on resident batch `b` as a CUDA graph
        (with cset: the step reads K1's outputs from it, prepared before each replay)."""
        if id(b) in self._graphs:
            return self._graphs[id(b)]
        self._ensure(b)
        if cset is None:
            cset = self._batch_set(b)  # the set step_resident prepares before each replay
        g = torch.cuda.CUDAGraph()
        lib = dev._lib.load()
        l0 = lib.dippm_launch_count()
        with torch.cuda.graph(g, pool=self._pool):
            self._step(b, global_graphs, cset=cset)
        hit = self._graphs[id(b)] = (g, lib.dippm_launch_count() - l0)
        self._keep.append(b)  # captured pointers must stay alive
        return hit

    def _native_ok(self, b: Batch) -> bool:
        eng = self.engine
        return (NATIVE_STEP and eng.arch == "sage" and eng.fused_head_ok(b.G)
                and eng.overlap_wgrad and not dev.HEAD_POOL and eng.cta_pair == 0 and eng.gemm_hook is None
                and _lib.call is _LIB_CALL and b.y is not None)

    def _native_for(self, b: Batch) -> NativeStep | None:
        """The native executor's plan for batch b (built or rebuilt to fit), or None when the
        step has to run the Python orchestration."""
        if not self._native_ok(b):
            return None
        ws, nat = self.ws, self._native
        if nat is None or nat.ws is not ws or not nat.fits(b):
            if nat is not None:
                if torch.cuda.is_current_stream_capturing() or self._graphs:
                    self._keep.append(nat)  # captured steps still point at its CSR buffers
                else:
                    torch.cuda.current_stream().synchronize()  # in-flight steps may still use them
            self._native = nat = NativeStep(self, max(b.E, 2 * ws.N, nat.E if nat is not None else 0))
        return nat

    def _prep(self, nat: NativeStep, b: Batch, cset: CsrBuffers, stream: torch.cuda.Stream,
              bad_out: torch.Tensor | None = None) -> None:
        """K1 of b into cset on `stream`, after the last step that read cset; the compute
        stream waits for it.  Issued before the step, it runs while the previous step still
        computes (the host is ahead of the device)."""
        if cset.free is not None:
            stream.wait_event(cset.free)
        nat.prep(b, cset, stream, bad_out)
        cset.ready.record(stream)
        torch.cuda.current_stream().wait_event(cset.ready)

    def _release(self, cset: CsrBuffers | None) -> None:
        if cset is not None:
            if cset.free is None:
                cset.free = torch.cuda.Event()
            cset.free.record(torch.cuda.current_stream())

    def _resident_prep(self, b: Batch) -> CsrBuffers | None:
        """K1 ahead of a resident batch's native step: a CSR set per batch when steps are
        captured (the graph holds its pointers), else a ring of two."""
        if not NATIVE_PREP or torch.cuda.is_current_stream_capturing():
            return None
        nat = self._native_for(b)
        if nat is None:
            return None
        if self.use_graphs:
            cset = self._batch_set(b)
        else:
            ring = self._csr_ring
            k = self._csr_next
            self._csr_next = 1 - k
            if ring[k] is None or not ring[k].fits(b):
                if ring[k] is not None and ring[k].free is not None:
                    ring[k].free.synchronize()
                ring[k] = CsrBuffers(max(b.N, self.ws.N), max(b.E, 2 * self.ws.N), max(b.G, self.ws.G),
                                     self.engine.device)
            cset = ring[k]
        ready = getattr(b, "_inputs_ready", None)  # the batch's own uploads (issued on the compute stream)
        if ready is None:
            ready = b._inputs_ready = torch.cuda.Event()
            ready.record(torch.cuda.current_stream())
        self._prep_stream.wait_event(ready)
        self._prep(nat, b, cset, self._prep_stream)
        return cset

    def _batch_set(self, b: Batch) -> CsrBuffers | None:
        """The resident batch's own CSR set when its captured step reads K1's outputs from one
        (None: the step runs K1 itself)."""
        if not (NATIVE_PREP and self.use_graphs) or self._native_for(b) is None:
            return None
        cset = getattr(b, "_csr_set", None)
        if cset is None or not cset.fits(b):
            cset = b._csr_set = CsrBuffers(b.N, b.E, b.G, self.engine.device)
        return cset

    def _step(self, b: Batch, global_graphs: int | None, slot: int | None = None,
              cset: CsrBuffers | None = None) -> bool:
        """One step; True if the native executor ran it (with `slot`: its loss and edge flag
        went to the device ring entry `slot` instead of the workspace; with `cset`: K1 already
        ran into it)."""
        eng, ws = self.engine, self.ws
        nat = self._native_for(b)
        if nat is not None:
            nat.sync_hparams(self)
            dp = self.allreduce is not None
            # data parallel: the global-batch denominator (gnn.py:402-404), then the native step up
            # to the final gradients, one all-reduce of the flat gradient, and Adam
            nat.plan.grad_den = float(global_graphs if global_graphs else b.G * self.world_size) if dp else 0.0
            if slot is None:
                nat.step(b, cset=cset, no_adam=dp)
            else:
                nat.step(b, self._loss_dev[slot].data_ptr(), self._bad_dev[slot:slot + 1],
                         graphed=NATIVE_GRAPHED and not dp, cset=cset, no_adam=dp)
            eng._uploaded = None
            ws.head_pending = None
            eng.launches += 20
            if dp:
                self.allreduce(eng.grads)  # sum of the per-rank gradient shares (NCCL on this stream)
                eng._t_advanced = True     # the step's head advanced t
                eng.adam_step(self.lr)
                eng.launches += 1
            eng._t_advanced = False  # the step's head advanced t and its Adam ran
            return True
        build_batch_csr(b)
        mode = 2 if self.dropout_p > 0 else 0
        eng.forward(b, ws, mask_mode=mode, dropout_p=self.dropout_p, seed=self.seed * 131 + self.rank,
                    predict=False, defer_head=True)
        den = 0.0
        if self.allreduce is not None:
            den = float(global_graphs if global_graphs else b.G * self.world_size)
        eng.loss(b, ws, self.delta, grad_den=den)
        keep = 1.0 / (1.0 - self.dropout_p) if mode else 1.0
        if self.allreduce is not None and hasattr(self.allreduce, "begin"):
            # two buckets: head + sage3 overlaps the layer-2/1 backward, the rest follows it
            split = {}

            def first_bucket(off):
                split["off"] = off
                self.allreduce.begin(eng.grads[off:])
            eng.backward(b, ws, keep_scale=keep, on_partial=first_bucket, advance_step=True)
            self.allreduce.begin(eng.grads[:split.get("off", eng.grads.numel())])
            self.allreduce.finish()
        else:
            eng.backward(b, ws, keep_scale=keep, advance_step=True)
            if self.allreduce is not None:
                self.allreduce(eng.grads)      # the one exchange: sum of per-rank gradient shares
        eng.adam_step(self.lr)
        return False

    def step_host(self, x, src, dst, graph_ptr, fs, y, edge_ptr=None, global_graphs: int | None = None) -> float:
        """End-to-end step from host (ideally pinned) buffers; returns the batch loss.

        edge_ptr [G+1] (edges grouped by graph, as collation produces) enables the
        per-graph CSR kernel; if omitted it is derived on the host when possible.
        global_graphs: the data-parallel batch size over all ranks (the gradient
        denominator); default: summed over the ranks with one small all-reduce."""
        return self.submit(x, src, dst, graph_ptr, fs, y, edge_ptr, global_graphs).loss()

    def submit(self, x, src, dst, graph_ptr, fs, y, edge_ptr=None, global_graphs: int | None = None) -> "StepHandle":
        """Asynchronous end-to-end step from host buffers (pipelined `step_host`).

        The batch is copied host->device on a side copy stream into one of two
        staging slots while the previous step still computes; the step then
        runs on the current stream and its loss is read back device->host into
        pinned memory.  Returns a StepHandle whose .loss() waits for that read.
        Steps stay in submission order (one compute stream), so the result is
        the same as calling step_host repeatedly.

        The batch is validated on the host first (edge endpoints inside their graph,
        ShapeMismatch otherwise); the handle's .loss() raises NonFinite for a non-finite
        loss (gnn.py:455-456) and ShapeMismatch if the device CSR build flagged an edge."""
        if edge_ptr is None:
            edge_ptr = dev.group_edges(np.asarray(src), np.asarray(dst), np.asarray(graph_ptr))
        arrays = [x, src, dst, graph_ptr, fs, y] + ([edge_ptr] if edge_ptr is not None else [])
        t = [torch.as_tensor(a) for a in arrays]
        G, N, E = t[3].numel() - 1, t[0].shape[0], t[1].numel()
        slots = self._slots
        if not slots or N > slots[0]["x"].shape[0] or E > slots[0]["src"].numel() or G + 1 > slots[0]["gp"].numel():
            torch.cuda.current_stream().synchronize()  # in-flight steps may still read the old slots
            self.reserve(max(N, self.ws.N if self.ws else 0), max(G, self.ws.G if self.ws else 0), max_edges=2 * E)
            slots = self._slots
        k = self._slot_next
        self._slot_next = 1 - k
        sl = slots[k]
        compute = torch.cuda.current_stream()
        views = [sl["x"][:N], sl["src"][:E], sl["dst"][:E], sl["gp"][:G + 1], sl["fs"][:G], sl["y"][:G],
                 sl["ep"][:G + 1]]
        b = Batch(G=G, N=N, E=E, x=views[0], src=views[1], dst=views[2], graph_ptr=views[3], fs=views[4], y=views[5],
                  h2d_bytes=sum(a.numel() * a.element_size() for a in t))
        if edge_ptr is not None:
            gp, ep = t[3].numpy(), np.asarray(edge_ptr)
            b.edge_ptr, b.max_nodes = views[6], int(np.diff(gp).max())
            b.max_edges = int(np.diff(ep).max()) if len(ep) > 1 else 0
        if global_graphs is None and self.allreduce is not None:
            from .dist import global_batch_size
            global_graphs = global_batch_size(G)  # ragged per-rank batches: the true global mean
        self._ensure(b)
        self.steps += 1
        j = self._loss_next
        self._loss_next = (j + 1) % len(self._loss_ring)
        host, flag = self._loss_ring[j], self._flag_ring[j]
        # native steps: K1 runs on the copy stream right behind this batch's copies, into the
        # slot's CSR set, so it overlaps the previous step
        nat = self._native_for(b) if NATIVE_PREP and not torch.cuda.is_current_stream_capturing() else None
        cset = None
        if nat is not None:
            cset = sl.get("csr")
            if cset is None or not cset.fits(b):
                cset = sl["csr"] = CsrBuffers(sl["x"].shape[0], max(sl["src"].numel(), E), sl["gp"].numel() - 1,
                                              self.engine.device)
        with torch.cuda.stream(self._copy_stream):
            self._copy_stream.wait_event(sl["free"])  # the step that last read this slot is done
            for d_, h in zip(views, t):
                d_.copy_(h, non_blocking=True)
            if cset is not None:
                nat.prep(b, cset, self._copy_stream, self._bad_dev[j:j + 1])
            sl["ready"].record(self._copy_stream)
        compute.wait_event(sl["ready"])
        native = self._step(b, global_graphs, slot=j, cset=cset)  # ragged shapes: host batches run eagerly
        sl["free"].record(compute)
        done = torch.cuda.Event()
        if native:  # loss / flag went to ring entry j: read back on the D2H stream, off the compute stream
            done.record(compute)
            self._d2h_stream.wait_event(done)
            with torch.cuda.stream(self._d2h_stream):
                host.copy_(self._loss_dev[j, :1], non_blocking=True)
                flag.copy_(self._bad_dev[j:j + 1], non_blocking=True)
                done = torch.cuda.Event()
                done.record(self._d2h_stream)
        else:
            host.copy_(self.ws.loss[:1], non_blocking=True)
            flag.copy_(b.bad[:1], non_blocking=True)
            done.record(compute)
        return StepHandle(done, host, flag)

    def sync_model(self):
        """Copy the device fp64 masters back into the host model's live arrays."""
        final = self.engine.get_params()
        for name, arr in self.model.param_items():
            arr[...] = final[name]
        return self.model


_LIB_CALL = _lib.call  # the unpatched library call (instrumented runs keep the Python step)


class StepHandle:
    """Result of BatchTrainer.submit: .loss() waits for the step's loss read-back."""

    def __init__(self, event, host, flag=None):
        self._event, self._host, self._flag = event, host, flag

    def done(self) -> bool:
        return self._event.query()

    def loss(self) -> float:
        self._event.synchronize()
        if self._flag is not None and int(self._flag[0]):
            raise ShapeMismatch("edge endpoint outside its graph's node range")
        v = float(self._host[0])
        if not math.isfinite(v):
            raise NonFinite("training loss is not finite")
        return v
