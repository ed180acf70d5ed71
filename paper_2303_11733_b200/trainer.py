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

import math

import numpy as np
import torch

from . import device as dev
from .device import Batch, Engine, Workspace, build_batch_csr
from .errors import NonFinite, ShapeMismatch


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

    def reserve(self, max_nodes: int, max_graphs: int, max_edges: int | None = None) -> None:
        """Preallocate the workspace (and host-batch staging) for batches up to this size."""
        self.ws = Workspace(self.engine, max_nodes, max_graphs, train=True)
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
        per-rank gradients is the global batch mean (gnn.py:402-404)."""
        self._ensure(b)
        self.steps += 1
        self.engine._uploaded = None  # the step moves the device parameters
        if not self.use_graphs:
            self._step(b, global_graphs)
            return
        # CUDA graphs: the trainer's first step runs eagerly (module load, kernel
        # attributes); afterwards each resident batch's step is captured once
        # and replayed.  Step-dependent values (Adam's t, the dropout stream)
        # live on the device, so replays advance them.
        hit = self._graphs.get(id(b))
        if hit is None:
            if not self._warm:
                self._step(b, global_graphs)
                self._warm = True
                return
            hit = self.capture(b, global_graphs)
        hit[0].replay()
        self.replayed_launches += hit[1]

    def capture(self, b: Batch, global_graphs: int | None = None):
        """Record (without executing) the training step on resident batch `b` as a CUDA graph."""
        if id(b) in self._graphs:
            return self._graphs[id(b)]
        self._ensure(b)
        g = torch.cuda.CUDAGraph()
        lib = dev._lib.load()
        l0 = lib.dippm_launch_count()
        with torch.cuda.graph(g, pool=self._pool):
            self._step(b, global_graphs)
        hit = self._graphs[id(b)] = (g, lib.dippm_launch_count() - l0)
        self._keep.append(b)  # captured pointers must stay alive
        return hit

    def _step(self, b: Batch, global_graphs: int | None) -> None:
        eng, ws = self.engine, self.ws
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
        with torch.cuda.stream(self._copy_stream):
            self._copy_stream.wait_event(sl["free"])  # the step that last read this slot is done
            views = [sl["x"][:N], sl["src"][:E], sl["dst"][:E], sl["gp"][:G + 1], sl["fs"][:G], sl["y"][:G],
                     sl["ep"][:G + 1]]
            for d_, h in zip(views, t):
                d_.copy_(h, non_blocking=True)
            sl["ready"].record(self._copy_stream)
        compute.wait_event(sl["ready"])
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
        self._step(b, global_graphs)  # ragged shapes: host batches run eagerly
        sl["free"].record(compute)
        j = self._loss_next
        self._loss_next = (j + 1) % len(self._loss_ring)
        host, flag = self._loss_ring[j], self._flag_ring[j]
        host.copy_(self.ws.loss[:1], non_blocking=True)
        flag.copy_(b.bad[:1], non_blocking=True)
        done = torch.cuda.Event()
        done.record(compute)
        return StepHandle(done, host, flag)

    def sync_model(self):
        """Copy the device fp64 masters back into the host model's live arrays."""
        final = self.engine.get_params()
        for name, arr in self.model.param_items():
            arr[...] = final[name]
        return self.model


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
