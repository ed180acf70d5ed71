#!/usr/bin/env python
"""DIPPM GraphSAGE training throughput on B200 (BASELINE.json metric, configs[1]).

Workload (configs[1]): one training epoch over a synthetic 10,508-graph
dataset shaped like the paper's corpus (N ~ U[270, 330] nodes, E/N ~ 1.33,
32-wide node rows, 5 static features), batch 256, hidden 512, Adam, dropout
0.05.  A "step" = one training step on one batch of 256 graphs: K1 CSR build
from the batch's edge list, 3 SAGE layers (K2 aggregation + K3 tcgen05 GEMM),
K4 pooling, K5 head, Huber loss, full backward, fused Adam, weight repack.

  value  graphs/s with the epoch's batches already resident in HBM
  e2e    graphs/s through the public batch-training call with HOST pinned
         batches: H2D of the batch + step + D2H of the loss inside the timing
  roofline  the dominant kernel family (tcgen05 GEMMs) vs measured peak
  cpu_baseline  the CPU oracle (numpy fp64 restatement of the reference,
         `oracle/`) on a bounded sample on this box's host cores

Multi-GPU (torchrun, one process per GPU): data parallel, weak scaling — each
rank trains on its own batch of 256 per step, gradients are summed with one
NCCL all-reduce (the path's only exchange) and averaged inside Adam.
Inputs per step exceed L2 (≈76.8k node rows, >150 MB of activations; the
epoch cycles through 41 distinct batches), so no explicit L2 flush is used.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "DIPPM graphs/sec (inference & training) at 1/2/4/8 B200; % of roofline"
DATA = "synthetic (generator B, seeded): paper-shaped 10,508-graph corpus, random-init weights"
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200, help="timed steps (~5 epochs of the 41-batch corpus)")
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                   help="gloo: multi-rank smoke runs (several ranks may share one GPU)")
    p.add_argument("--dtype", choices=["bf16", "fp32"], default="bf16")
    p.add_argument("--graphs", type=int, default=10508)
    p.add_argument("--batch", type=int, default=256)
    p.add_argument("--hidden", type=int, default=512)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-graphs", action="store_true", help="launch the training step eagerly (no CUDA graph)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-steps", type=int, default=16, help="CPU baseline sample: steps of one batch each")
    p.add_argument("--clock-ms", type=int, default=10, help="NVML sampling interval during timing")
    p.add_argument("--no-clocks", action="store_true")
    p.add_argument("--no-infer", action="store_true", help="skip the configs[2]-[4] sweeps")
    p.add_argument("--no-fp32", action="store_true", help="skip the fp32-mode training line")
    p.add_argument("--no-cfg0", action="store_true", help="skip the configs[0] fp32 inference line")
    p.add_argument("--infer-batch", type=int, default=4096)
    p.add_argument("--infer-batches", type=int, default=8, help="configs[2] batches per rank")
    return p.parse_args()


def peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        return d, "measured (MEASURED_PEAKS.json)"
    return FALLBACK_PEAKS, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)

class ClockSampler:
    """SM clock + throttle reasons sampled in-process through NVML (pynvml) on a
    background thread during the timed region.  (Spawning `nvidia-smi -lms`
    instead was measured to stall the GPU work it is observing.)"""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, gpu_index: int, interval_ms: int = 50):
        self.gpu, self.interval = gpu_index, interval_ms
        self.samples, self.active, self.stop_flag, self.thread, self.h = [], False, False, None, None

    def start(self):
        try:
            import threading

            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 - report "not sampled" instead of failing the bench
            self.h = None
            return

        def loop():
            while not self.stop_flag:
                if self.active:
                    try:
                        c = self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM)
                        r = self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                        self.samples.append((c, r))
                    except Exception:  # noqa: BLE001
                        pass
                time.sleep(self.interval / 1000.0)

        self.thread = threading.Thread(target=loop, daemon=True)
        self.thread.start()

    def wait_first_sample(self):
        pass

    def mark(self):
        self.samples.clear()
        self.active = True

    def stop(self):
        self.active = False
        self.stop_flag = True
        if self.thread is not None:
            self.thread.join(timeout=2)
        if self.h is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml not sampled"]}
        reasons = sorted({name for _, r in self.samples for bit, name in self.REASONS.items() if r & bit})
        sm = [c for c, _ in self.samples]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(sm), "source": "nvml in-process"}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle (fp64 numpy restatement of gnn.backward + Adam)

_SHM = {}


def _cpu_worker_init(shm_name, shapes, hidden):
    from multiprocessing import shared_memory
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
    shm = shared_memory.SharedMemory(name=shm_name)
    _SHM["shm"] = shm
    flat = np.ndarray((sum(int(np.prod(s)) for _, s in shapes),), dtype=np.float64, buffer=shm.buf)
    params, off = {}, 0
    for name, s in shapes:
        n = int(np.prod(s))
        params[name] = flat[off:off + n].reshape(s)
        off += n
    _SHM["params"] = params
    _SHM["hidden"] = hidden


def _cpu_worker_grads(args):
    from oracle import dippm_oracle as O
    ids, norm = args  # graph ids into the dataset the worker inherited at fork time
    recs = [(r.encoding.num_nodes, r.encoding.edges, r.encoding.features, r.fs.as_vector, r.target.as_array)
            for r in _SHM["ds"].records(ids)]
    loss, grads = O.backward(_SHM["params"], norm, recs, hidden=_SHM["hidden"])
    n = len(recs)
    return loss * n, {k: g * n for k, g in grads.items()}, n


class CpuOracleTrainer:
    """Batch-protocol CPU training step (gnn.backward over a batch of records + 15 Adam
    updates, the oracle's fp64 numpy restatement) on `procs` worker processes with 1 BLAS
    thread each; parameters live in shared memory, the pool is created once."""

    def __init__(self, ds, hidden, procs, seed=0):
        import multiprocessing as mp
        from multiprocessing import shared_memory
        from oracle import dippm_oracle as O
        self.O, self.ds, self.procs = O, ds, procs
        rng = np.random.default_rng(seed)
        self.rng = rng
        params = O.init_params(hidden, rng)
        self.shapes = [(k, params[k].shape) for k in O.SAGE_PARAM_NAMES]
        total = sum(int(np.prod(s)) for _, s in self.shapes)
        self.shm = shared_memory.SharedMemory(create=True, size=total * 8)
        flat = np.ndarray((total,), dtype=np.float64, buffer=self.shm.buf)
        self.views, off = {}, 0
        for k, s in self.shapes:
            n = int(np.prod(s))
            flat[off:off + n] = params[k].ravel()
            self.views[k] = flat[off:off + n].reshape(s)
            off += n
        self.norm = O.normalizer_fit(ds.y.astype(np.float64), ds.fs.astype(np.float64))
        self.state = {k: (np.zeros(s), np.zeros(s)) for k, s in self.shapes}
        self.t = 0
        _SHM["ds"] = ds  # inherited by the forked workers: steps ship graph ids, not arrays
        self.pool = mp.get_context("fork").Pool(procs, initializer=_cpu_worker_init,
                                                initargs=(self.shm.name, self.shapes, hidden))

    def records(self, n):
        return self.rng.choice(self.ds.num_graphs, n, replace=False)

    def step(self, recs):
        parts = [(recs[i::self.procs], self.norm) for i in range(self.procs) if len(recs[i::self.procs])]
        out = self.pool.map(_cpu_worker_grads, parts)
        n = sum(o[2] for o in out)
        grads = {k: sum(o[1][k] for o in out) / n for k, _ in self.shapes}
        self.t += 1
        for k, _ in self.shapes:
            m, v = self.state[k]
            self.views[k][...] = self.O.adam_step(self.views[k], grads[k], m, v, self.t)

    def close(self):
        self.pool.close()
        self.pool.join()
        self.shm.close()
        self.shm.unlink()


def cpu_baseline(ds, hidden, batch, steps, procs, seed=0):
    """`steps` CPU steps of `batch` graphs; returns (graphs/s, seconds)."""
    tr = CpuOracleTrainer(ds, hidden, procs, seed)
    try:
        batches = [tr.records(batch) for _ in range(steps)]
        tr.step(batches[0][:procs])  # warm the workers
        t0 = time.perf_counter()
        for recs in batches:
            tr.step(recs)
        dt = time.perf_counter() - t0
    finally:
        tr.close()
    return steps * batch / dt, dt


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def config_dict(args, world):
    return {"workload": "configs[1]: GraphSAGE training epoch, synthetic 10,508-graph paper-shaped corpus, "
                        "batch 256/rank, Adam",
            "graphs": args.graphs, "batch_per_rank": args.batch, "global_batch": args.batch * world,
            "hidden": args.hidden, "nodes_per_graph": "U[270,330]", "edges_per_node": 1.33,
            "parallelism": f"dp{world}", "l2": "inputs larger than L2 (no flush)",
            "launch": "eager" if getattr(args, "no_graphs", False) or world > 1 else "cuda_graph (one per resident batch)",
            "collective": f"{getattr(args, 'dist_backend', 'nccl')} all-reduce of the fp32 gradient (6.4 MB) per step, "
                          "2 buckets, head+sage3 overlapped with the layer-2/1 backward"
            if world > 1 else None}


# ---------------------------------------------------------------------------

def run_reference(args, rank, world, budget_s=150.0):
    """Reference arm: the CPU port of the reference's path (the oracle: fp64 numpy
    gnn.backward + Adam, batch protocol) on all host cores, same config and metric.
    Warm-up steps are untimed; timed steps run until --steps are done or the time budget
    is spent (full 256-graph steps; the sample actually timed is stated)."""
    if rank != 0:
        return
    from paper_2303_11733_b200.synth import make_dataset
    ds = make_dataset(args.graphs, seed=2)
    procs = host_cores()
    tr = CpuOracleTrainer(ds, args.hidden, procs, seed=100)
    try:
        for _ in range(args.warmup):
            tr.step(tr.records(args.batch))
        done, total = 0, 0.0
        while done < args.steps and total < budget_s:
            recs = tr.records(args.batch)
            t0 = time.perf_counter()
            tr.step(recs)
            total += time.perf_counter() - t0
            done += 1
    finally:
        tr.close()
    value = done * args.batch / total
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "graphs/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * total / done,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": DATA, "config": dict(config_dict(args, world), arm="CPU reference port on rank 0 (all host cores); other ranks idle"),
            "cpu_baseline": {"value": value, "unit": "graphs/s", "cores": procs, "kind": "port",
                             "sample": f"{done} of {args.steps} timed steps x {args.batch} graphs (time budget "
                                       f"{budget_s:.0f} s), oracle gnn.backward + Adam (fp64 numpy), {procs} procs "
                                       f"x 1 BLAS thread, {cpu_model()}"},
            "e2e": {"value": value, "unit": "graphs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def inference_sweep(args, rank, world, lib):
    """configs[2]: batched predict (CSR + forward + de-normalise + MIG pick) over ONE corpus of
    world x infer_steps x infer_batch graphs (weak scaling: a fixed share per rank), sharded
    over the ranks by node count (dist.shard_by_nodes, contiguous graph ranges, no collective
    in the timed loop); each rank runs its share in batches of ~infer_batch graphs, graphs/s
    over all ranks from the max-over-ranks device time; then the (y, MIG) predictions of all
    graphs are collected on every rank (dist.gather_predictions, 16 B/graph), timed apart.
    bf16 twice: raw picks, and with the fp32 re-score of the graphs whose bf16 memory lies
    within the bf16 tolerance of a pick boundary (the bit-exact-pick path)."""
    import torch
    import torch.distributed as dist
    from paper_2303_11733_b200 import gnn
    from paper_2303_11733_b200 import device as dev
    from paper_2303_11733_b200.device import Engine, Workspace, build_batch_csr, upload_batch
    from paper_2303_11733_b200.dist import gather_predictions, shard_by_nodes
    from paper_2303_11733_b200.synth import make_dataset, node_counts

    per_rank = args.infer_batch * args.infer_batches
    total = per_rank * world
    counts = node_counts(total, np.random.default_rng(3))          # the corpus' node counts
    a, b_ = shard_by_nodes(counts, world)[rank]                    # this rank's contiguous share
    ds = make_dataset(b_ - a, seed=1000 + rank, nodes=counts[a:b_])  # its graphs (seeded per shard)
    norm = gnn.Normalizer.fit(ds.y.astype(np.float64), ds.fs.astype(np.float64))
    norm.y_mean[1], norm.y_std[1] = 20000.0, 13000.0  # memory spread over the MIG profiles
    model = gnn.create_model(hidden=args.hidden, seed=0, normalizer=norm)
    nb = max(1, -(-(b_ - a) // args.infer_batch))
    batches = [upload_batch(*ds.collate(np.arange(i * (b_ - a) // nb, (i + 1) * (b_ - a) // nb)),
                            device="cuda", build_csr=False) for i in range(nb)]
    out = {"workload": f"configs[2]: predict + MIG over a {total}-graph corpus sharded by node count over "
                       f"{world} rank(s) ({b_ - a} graphs on rank {rank}), batches of ~{args.infer_batch}, "
                       f"hidden {args.hidden}", "scaling": "weak", "graphs_total": total,
           "shard": "dist.shard_by_nodes (contiguous, balanced by nodes)"}
    eng32 = None
    for mode in ("bf16", "bf16_mig_exact", "fp32"):
        prec = "fp32" if mode == "fp32" else "bf16"
        eng = Engine(args.hidden, prec)
        eng.set_params(model.param_items(), norm)
        if mode == "bf16_mig_exact" and eng32 is None:
            eng32 = Engine(args.hidden, "fp32")
            eng32.set_params(model.param_items(), norm)
        ws = Workspace(eng, max(b.N for b in batches), max(b.G for b in batches), train=False)
        holder = type("Slots", (), {})()
        band = dev.BF16_MIG_BAND * float(norm.y_std[1])
        rescored = [0]
        ys, migs = [], []

        def step(i, keep=False):
            bt = batches[i % nb]
            build_batch_csr(bt)
            eng.forward(bt, ws, predict=True)
            if mode == "bf16_mig_exact":
                rescored[0] += dev.mig_band_rescore(eng32, bt, ws, band, holder)
            if keep:
                ys.append(ws.y_pred[:bt.G].clone())
                migs.append(ws.mig[:bt.G].clone())

        timer = GemmTimer()
        for i in range(max(3, nb)):  # every batch once: workspace growth and first launches stay untimed
            step(i)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        sampler = ClockSampler(int(os.environ.get("LOCAL_RANK", 0)), args.clock_ms)
        if not args.no_clocks:
            sampler.start()
        sampler.mark()
        rescored[0] = 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(nb):
            step(i, keep=True)
        e1.record()
        torch.cuda.synchronize()
        clocks = sampler.stop()
        ms = max_over_ranks(e0.elapsed_time(e1), world)
        t0 = time.perf_counter()
        y_all, mig_all = gather_predictions(torch.cat(ys), torch.cat(migs))
        torch.cuda.synchronize()
        t_gather = time.perf_counter() - t0
        assert y_all.shape[0] == total, (y_all.shape, total)
        entry = {"graphs_per_s": total / (ms / 1000.0), "ms_per_batch": ms / nb, "batches_per_rank": nb,
                 "clocks": clocks, "gather_ms": 1000 * t_gather,
                 "mig_code_counts": {str(c): int((mig_all == c).sum()) for c in (-1, 0, 1, 2, 3)}}
        if mode == "bf16_mig_exact":
            n_res = torch.tensor([rescored[0]], dtype=torch.int64, device="cuda")
            if world > 1:
                dist.all_reduce(n_res)
            entry["rescored_fp32"] = int(n_res.item())
            entry["rescored_frac"] = int(n_res.item()) / total
            entry["band_mb"] = band
        if mode != "bf16_mig_exact":
            eng.gemm_hook = timer
            for i in range(nb):
                step(i)
            eng.gemm_hook = None
            g_flops, g_ms, _ = timer.summary()
            entry.update(gemm_tflops=g_flops / (g_ms / 1000.0) / 1e12, gemm_share=g_ms / ms)
        out[mode] = entry
        del ws, eng
        torch.cuda.empty_cache()
    return out


def max_over_ranks(ms, world):
    """Device time of the slowest rank (the job's time)."""
    if world == 1:
        return ms
    import torch
    import torch.distributed as dist
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def train_large_graph_skew(args, rank, world, per_rank=32, batches=8, steps=40):
    """configs[3] per GPU: data-parallel training batches of 32 graphs per rank whose node counts
    are log-uniform on [12, 5000] (transformer-sized graphs mixed with tiny ones, SURVEY §8d
    cfg4); resident batches, CUDA-graph steps at N=1 (eager + the bucketed all-reduce at N>1),
    max-over-ranks device time, graphs/s over all ranks."""
    import torch
    import torch.distributed as dist
    from paper_2303_11733_b200 import gnn
    from paper_2303_11733_b200.device import upload_batch
    from paper_2303_11733_b200.dist import OverlappedAllReduce
    from paper_2303_11733_b200.synth import make_dataset
    rng = np.random.default_rng(40 + rank)
    n = np.exp(rng.uniform(np.log(12), np.log(5000), per_rank * batches)).astype(np.int64)
    ds = make_dataset(len(n), seed=40 + rank, nodes=n)
    norm = gnn.Normalizer.fit(ds.y.astype(np.float64), ds.fs.astype(np.float64))
    model = gnn.create_model(hidden=args.hidden, seed=0, normalizer=norm)
    from paper_2303_11733_b200.trainer import BatchTrainer
    tr = BatchTrainer(model, precision=args.dtype, lr=gnn.DEFAULT_LEARNING_RATE, seed=3,
                      allreduce=OverlappedAllReduce() if world > 1 else None, world_size=world, rank=rank,
                      use_graphs=world == 1)
    order = np.argsort(rng.random(len(n)))
    res = [upload_batch(*ds.collate(order[i * per_rank:(i + 1) * per_rank]), device="cuda", build_csr=False)
           for i in range(batches)]
    tr.reserve(max(b.N for b in res), per_rank)
    for i in range(3):
        tr.step_resident(res[i % batches])
    if tr.use_graphs:
        for b in res:
            tr.capture(b)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(steps):
        tr.step_resident(res[i % batches])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    nodes = [b.N for b in res]
    return {"workload": f"configs[3]: DP training, {per_rank} graphs/rank/step, node counts log-uniform on "
                        f"[12, 5000] (up to {int(max(ds.n))} nodes), hidden {args.hidden}, Adam",
            "graphs_per_s": steps * per_rank * world / (ms / 1000.0), "ms_per_step": ms / steps,
            "nodes_per_step_mean": float(np.mean(nodes)), "scaling": "weak"}


def predict_from_json(args, rank, world, docs_per_batch=4096, batches=2):
    """configs[4]: end-to-end predict + MIG pick from graph JSON documents with
    power-law operator counts (N in [12, 5000], alpha 1.5): native multi-threaded
    parse + shape inference + featurisation (libdippm_host.so), H2D, CSR, bf16
    forward, de-normalise + MIG on device, D2H of y and the MIG codes.  Wall
    clock of one predict_documents call over `batches` chunks (host work is part of
    the path; featurisation of chunk k+1 overlaps chunk k's device pass), documents/s
    over all ranks, with the two halves also timed alone."""
    import torch
    from paper_2303_11733_b200 import featurize as F
    from paper_2303_11733_b200 import gnn
    from paper_2303_11733_b200.synth import make_graph_documents
    docs = [d.encode() for d in make_graph_documents(docs_per_batch * batches, seed=50 + rank)]
    fb0 = F.featurize_documents(docs[:docs_per_batch])
    # normaliser spreading predicted memory over 0-45,000 MB so every MIG profile (and None) occurs
    norm = gnn.Normalizer(np.array([5.0, 74000.0, 2.0]), np.array([3.0, 150000.0, 1.0]),
                          fb0.fs_vectors().mean(0), fb0.fs_vectors().std(0) + 1e-3)
    model = gnn.create_model(hidden=args.hidden, seed=0, normalizer=norm)
    # warm: engine, kernels, and the pinned staging buffers of both pipeline slots (torch's
    # caching host allocator keeps them; a serving process pays the allocation once)
    F.predict_documents(model, docs, precision="bf16", chunk=docs_per_batch)
    torch.cuda.synchronize()
    n_docs = docs_per_batch * batches
    # the components alone: featurise every chunk, then the device half on the last one
    t0 = time.perf_counter()
    for k in range(batches):
        fb = F.featurize_documents(docs[k * docs_per_batch:(k + 1) * docs_per_batch])
    t_feat = time.perf_counter() - t0
    t0 = time.perf_counter()
    F.predict_featurized(model, fb, precision="bf16")
    t_dev = (time.perf_counter() - t0) * batches
    # the path itself: one call, featurisation of chunk k+1 overlapped with chunk k's device pass
    t0 = time.perf_counter()
    _, codes, _ = F.predict_documents(model, docs, precision="bf16", chunk=docs_per_batch)
    t_all = time.perf_counter() - t0
    return {"workload": f"configs[4]: graph JSON -> native featurise -> bf16 predict + MIG, {n_docs} "
                        f"power-law graphs per call in chunks of {docs_per_batch}, hidden {args.hidden}",
            "docs_per_s": n_docs * world / t_all, "featurise_docs_per_s": n_docs / t_feat,
            "device_docs_per_s": n_docs / t_dev, "pipelined_chunks": batches,
            "mean_operator_nodes": float(fb0.n.mean()), "host_threads": os.cpu_count(),
            "mig_code_counts": {str(c): int((codes == c).sum()) for c in (-1, 0, 1, 2, 3)}}


class GemmTimer:
    """CUDA-event pairs around each tensor-core GEMM launch (on the launching stream)."""

    def __init__(self):
        import torch
        self.torch = torch
        self.recs = []

    def __call__(self, phase, flops):
        ev = self.torch.cuda.Event(enable_timing=True)
        ev.record()
        if phase == "pre":
            self.recs.append([ev, None, flops])
        else:
            self.recs[-1][1] = ev

    def summary(self):
        self.torch.cuda.synchronize()
        ms = [a.elapsed_time(b) for a, b, _ in self.recs]
        flops = [f for _, _, f in self.recs]
        return sum(flops), sum(ms), len(ms)

    def classes(self, steps, big=2e10):
        """Per-step split: the layer-2/3 SAGE GEMMs (M = nodes, K >= 512: >= 20 GFLOP each) vs the
        rest (layer-1 K = 64 and weight-gradient GEMMs, the 256-row head)."""
        self.torch.cuda.synchronize()
        out = {}
        for name, sel in (("sage_layers_2_3", lambda f: f >= big), ("layer1_and_head", lambda f: f < big)):
            rs = [(a.elapsed_time(b), f) for a, b, f in self.recs if sel(f)]
            t, f = sum(r[0] for r in rs), sum(r[1] for r in rs)
            out[name] = {"launches_per_step": len(rs) / steps, "us_per_step": 1e3 * t / steps,
                         "tflop_per_step": f / steps / 1e12, "tflops": f / (t / 1e3) / 1e12 if t else None}
        return out


class KernelTimer:
    """CUDA events around the HBM-bound kernels of a step (K1 CSR, K2 aggregation, K2^T /
    readout backward, K4 pool combine), recorded on the launching stream by wrapping the
    package's C-ABI call helper; each launch is tagged with its algorithmic bytes
     computed from the batch shape."""

    def __init__(self, lib_mod, hp, elem):
        import torch
        self.torch, self.lib_mod, self.hp, self.elem = torch, lib_mod, hp, elem
        self.recs = []
        self.batch = None  # (N, E, G) of the step being timed
        self._orig = None

    def bytes_for(self, name, args):
        N, E, G = self.batch
        hp, s = self.hp, self.elem
        if name in ("dippm_build_csr_grouped", "dippm_build_csr"):
            # read src/dst int64; write rowptr, col, deg, inv_deg, t_rowptr, t_col, node_graph
            return "K1_csr", 16 * E + 8 * E + 8 * (N + 1) + 12 * N
        if name == "dippm_sage_aggregate":
            d = int(args[4])
            if d == 32:  # layer 1: fp32 X gathered and copied, [X | agg X] written in the compute dtype
                return "K2_aggregate_l1", E * d * 4 + N * d * 4 + 2 * N * d * s + 4 * (N + 1 + E) + 4 * N
            return "K2_aggregate_l23", E * d * s + N * d * s + 4 * (N + 1 + E) + 4 * N
        if name == "dippm_sage_aggregate_t":
            return "K2T_aggregate_t", E * hp * s + 2 * N * hp * s + 4 * (N + 1 + E) + 4 * N
        if name == "dippm_readout_aggregate_t":
            # du [G, hp] fp32, h3 ReLU bits, CSR^T; writes [dz3 | agg^T dz3]
            return "K2T_readout", G * hp * 4 + N * hp // 8 + 2 * N * hp * s + 4 * (N + 1 + E) + 4 * N
        if name == "dippm_pool_combine":
            return "K4_pool_combine", (2 * ((N + 31) // 32) + G) * hp * 4 + G * (hp + 64) * s
        return None, 0

    def install(self):
        orig = self._orig = self.lib_mod.call
        torch = self.torch

        def call(name, *args):
            tag, nbytes = self.bytes_for(name, args) if self.batch is not None else (None, 0)
            if tag is None:
                return orig(name, *args)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            r = orig(name, *args)
            e1.record()
            self.recs.append((tag, nbytes, e0, e1))
            return r
        self.lib_mod.call = call

    def uninstall(self):
        if self._orig is not None:
            self.lib_mod.call = self._orig

    def summary(self, peak_gbs):
        self.torch.cuda.synchronize()
        agg = {}
        for tag, nb, e0, e1 in self.recs:
            a = agg.setdefault(tag, [0, 0.0, 0])
            a[0] += nb
            a[1] += e0.elapsed_time(e1)
            a[2] += 1
        out = {}
        for tag, (nb, ms, n) in sorted(agg.items()):
            gbs = nb / (ms / 1000.0) / 1e9
            out[tag] = {"launches": n, "us_per_launch": 1000 * ms / n, "algorithmic_bytes_per_launch": nb / n,
                        "achieved_gbs": gbs, "frac": gbs / peak_gbs}
        return out


def maybe_spawn(args):
    """`python bench.py --gpus N` (N > 1) without torchrun: re-exec under torch.distributed.run
    with one process per GPU (rendezvous on 127.0.0.1); rank 0 prints the JSON line."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def train_throughput(trainer, resident, steps, warmup, world, use_graphs, sampler=None):
    """Time `steps` resident training steps (after `warmup`), max over ranks; (ms, launches)."""
    import torch
    import torch.distributed as dist
    lib = trainer.engine and __import__("paper_2303_11733_b200._lib", fromlist=["load"]).load()
    nb = len(resident)
    for i in range(warmup):
        trainer.step_resident(resident[i % nb])
    if use_graphs:  # setup: record each resident batch's step (capture executes nothing)
        for b in resident:
            trainer.capture(b)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    if sampler is not None:
        sampler.mark()
    l0 = lib.dippm_launch_count() + trainer.replayed_launches
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    for i in range(steps):
        trainer.step_resident(resident[(warmup + i) % nb])
    end.record()
    torch.cuda.synchronize()
    launches = lib.dippm_launch_count() + trainer.replayed_launches - l0
    return max_over_ranks(start.elapsed_time(end), world), launches


def configs0_inference(args, rank, procs):
    """configs[0]: fp32 inference of one 256-graph batch (~300 nodes/graph) — the reference's
    own CPU-runnable case.  Device-resident graphs/s, end-to-end graphs/s through
    gnn.predict_batch (host encodings in, y and MIG picks out), and the CPU oracle on the
    same 256 graphs with one process per core."""
    import torch
    from paper_2303_11733_b200 import gnn
    from paper_2303_11733_b200.device import Engine, Workspace, build_batch_csr, upload_batch
    from paper_2303_11733_b200.synth import make_dataset
    ds = make_dataset(256, seed=1)
    norm = gnn.Normalizer.fit(ds.y.astype(np.float64), ds.fs.astype(np.float64))
    model = gnn.create_model(hidden=args.hidden, seed=0, normalizer=norm)
    eng = Engine(args.hidden, "fp32")
    eng.set_params(model.param_items(), norm)
    b = upload_batch(*ds.collate(np.arange(256)), device="cuda", build_csr=False)
    ws = Workspace(eng, b.N, b.G, train=False)
    for _ in range(3):
        build_batch_csr(b)
        eng.forward(b, ws)
    torch.cuda.synchronize()
    reps = 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        build_batch_csr(b)
        eng.forward(b, ws)
    e1.record()
    torch.cuda.synchronize()
    dev_ms = e0.elapsed_time(e1) / reps
    recs = ds.records(range(256))
    encs, fss = [r.encoding for r in recs], [r.fs for r in recs]
    gnn.predict_batch(model, encs, fss, precision="fp32")
    t0 = time.perf_counter()
    for _ in range(5):
        gnn.predict_batch(model, encs, fss, precision="fp32")
    e2e_s = (time.perf_counter() - t0) / 5
    out = {"workload": "configs[0]: fp32 inference, one batch of 256 synthetic graphs (N ~ U[270,330]), "
                       f"hidden {args.hidden}", "dtype": "fp32 (3-pass tf32 tensor cores)",
           "graphs_per_s": 256 / (dev_ms / 1000.0), "ms_per_batch": dev_ms,
           "e2e_graphs_per_s": 256 / e2e_s, "e2e": "gnn.predict_batch from host encodings (collate, H2D, CSR, "
                                                   "forward, de-normalise, MIG, D2H), wall clock"}
    if rank == 0 and not args.no_cpu_baseline:
        import multiprocessing as mp
        from oracle import dippm_oracle as O
        params = {k: np.array(v) for k, v in model.param_items()}
        nd = {"y_mean": norm.y_mean, "y_std": norm.y_std, "fs_mean": norm.fs_mean, "fs_std": norm.fs_std}
        orecs = [(r.encoding.num_nodes, r.encoding.edges, r.encoding.features, r.fs.as_vector) for r in recs]
        _SHM["c0"] = (params, nd, orecs)
        with mp.get_context("fork").Pool(procs, initializer=_limit_blas) as pool:
            t0 = time.perf_counter()
            ref = pool.map(_c0_predict, range(256), chunksize=max(1, 256 // (4 * procs)))
            cpu_s = time.perf_counter() - t0
        y, _ = gnn.predict_batch(model, encs, fss, precision="fp32")
        ref = np.array(ref)
        out["cpu_baseline"] = {"value": 256 / cpu_s, "unit": "graphs/s", "cores": procs, "kind": "port",
                               "sample": f"the same 256 graphs: oracle predict (fp64 numpy), {procs} procs x 1 BLAS "
                                         f"thread, {cpu_model()}"}
        out["max_rel_err_vs_oracle"] = float(np.max(np.abs(y - ref) / np.abs(ref)))
    return out


def _limit_blas():
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)


def _c0_predict(i):
    from oracle import dippm_oracle as O
    params, nd, orecs = _SHM["c0"]
    return O.predict(params, nd, *orecs[i])


def main():
    args = parse_args()
    maybe_spawn(args)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    if args.dist_backend == "nccl" and world > torch.cuda.device_count():
        raise SystemExit(f"bench.py: {world} NCCL ranks but {torch.cuda.device_count()} visible GPUs")
    local = local % max(torch.cuda.device_count(), 1)  # ranks may share a GPU in gloo smoke runs
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    from paper_2303_11733_b200 import _lib, gnn
    from paper_2303_11733_b200.device import upload_batch
    from paper_2303_11733_b200.dist import OverlappedAllReduce
    from paper_2303_11733_b200.synth import make_dataset
    from paper_2303_11733_b200.trainer import BatchTrainer

    lib = _lib.load()
    ds = make_dataset(args.graphs, seed=2)
    rng = np.random.default_rng(7)
    perm = rng.permutation(ds.num_graphs)[rank::world]
    nb = len(perm) // args.batch
    batches_host = [ds.collate(perm[i * args.batch:(i + 1) * args.batch]) for i in range(nb)]
    norm = gnn.Normalizer.fit(ds.y.astype(np.float64), ds.fs.astype(np.float64))
    model = gnn.create_model(hidden=args.hidden, seed=0, normalizer=norm)
    use_graphs = not args.no_graphs and world == 1  # the all-reduce stays outside graph capture

    def make_trainer(precision):
        return BatchTrainer(model, precision=precision, lr=gnn.DEFAULT_LEARNING_RATE, seed=11,
                            allreduce=OverlappedAllReduce() if world > 1 else None, world_size=world, rank=rank,
                            use_graphs=use_graphs)

    trainer = make_trainer(args.dtype)
    eng = trainer.engine
    # resident epoch: every batch collated in HBM before timing (CSR is rebuilt each step)
    resident = [upload_batch(*b, device=eng.device, build_csr=False) for b in batches_host]
    trainer.reserve(max(b.N for b in resident), args.batch)
    torch.cuda.synchronize()

    sampler = ClockSampler(local, args.clock_ms)
    if not args.no_clocks:
        sampler.start()
    t_wall = time.perf_counter()
    ms, launches = train_throughput(trainer, resident, args.steps, args.warmup, world, use_graphs, sampler)
    wall = time.perf_counter() - t_wall
    clocks = sampler.stop()
    graphs = args.steps * args.batch * world
    value = graphs / (ms / 1000.0)

    # roofline pass: the same steps launched eagerly on one stream, CUDA events around every
    # tcgen05 GEMM (eng.gemm_hook) and every HBM-bound kernel (KernelTimer)
    pk, pk_src = peaks()
    elem = 2 if args.dtype == "bf16" else 8  # fp32 mode stores activations as two fp32 planes
    ktimer = KernelTimer(_lib, eng.L.hp, elem)
    timer = GemmTimer()
    eng.gemm_hook = timer
    trainer.use_graphs = False
    overlap, eng.overlap_wgrad = eng.overlap_wgrad, False  # each kernel timed alone on one stream
    ktimer.install()
    try:
        for i in range(args.steps):
            b = resident[(args.warmup + args.steps + i) % nb]
            ktimer.batch = (b.N, b.E, b.G)
            trainer.step_resident(b)
    finally:
        ktimer.uninstall()
        eng.gemm_hook = None
        eng.overlap_wgrad = overlap
        trainer.use_graphs = use_graphs
    g_flops, g_ms, g_n = timer.summary()
    # each GEMM is timed alone inside a short eager pass: the burst peak is the denominator
    peak_tf = pk["bf16_tflops"] if args.dtype == "bf16" else pk["bf16_tflops"] / 6.0
    achieved = g_flops / (g_ms / 1000.0) / 1e12
    step_flops = g_flops / args.steps
    traffic = None
    prof = ROOT / "profiles" / "ncu_summary.json"
    if prof.exists():
        traffic = json.loads(prof.read_text()).get(f"gemm_dram_bytes_per_launch_{args.dtype}")
    hbm = ktimer.summary(pk["hbm_gbs"])

    # e2e: public batch-training call with host pinned batches
    e2e = None
    if not args.no_e2e:
        from paper_2303_11733_b200.device import group_edges
        # (static features and targets in float64, the host layout collate_host produces)
        pinned = [[torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
                   for a in (*b[:4], b[4].astype(np.float64), b[5].astype(np.float64), group_edges(b[1], b[2], b[3]))]
                  for b in batches_host]
        h2d = sum(sum(t.numel() * t.element_size() for t in b) for b in pinned) / len(pinned)
        gg = args.batch * world  # uniform per-rank batches: the global denominator is known
        for i in range(2):
            trainer.step_host(*pinned[i % nb], global_graphs=gg)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        # pipelined public call: H2D of batch i+1 overlaps step i; every step's loss is
        # read back to the host (handles consumed at most 16 steps behind)
        pending, losses = [], []
        for i in range(args.steps):
            pending.append(trainer.submit(*pinned[(args.warmup + i) % nb], global_graphs=gg))
            if len(pending) > 16:
                losses.append(pending.pop(0).loss())
        losses += [h.loss() for h in pending]
        e1.record()
        torch.cuda.synchronize()
        assert len(losses) == args.steps and all(np.isfinite(losses))
        ems = max_over_ranks(e0.elapsed_time(e1), world)
        e2e = {"value": graphs / (ems / 1000.0), "unit": "graphs/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": 8 + 4, "api": "BatchTrainer.submit (pinned host batch -> loss on host)"}

    # the parity-grade fp32 mode on the same workload (bounded sample of steps)
    train_fp32 = None
    if not args.no_fp32 and args.dtype == "bf16":
        tr32 = make_trainer("fp32")
        tr32.reserve(max(b.N for b in resident), args.batch)
        k = max(4, args.steps // 10)
        ms32, _ = train_throughput(tr32, resident, k, 3, world, use_graphs)
        train_fp32 = {"graphs_per_s": k * args.batch * world / (ms32 / 1000.0), "ms_per_step": ms32 / k,
                      "steps": k, "dtype": "fp32 (3-pass tf32 tensor cores, fp64 Adam masters)"}
        del tr32
        torch.cuda.empty_cache()

    infer = None
    if not args.no_infer:
        infer = inference_sweep(args, rank, world, lib)
        infer["predict_from_json"] = predict_from_json(args, rank, world)
        infer["train_large_graph_skew"] = train_large_graph_skew(args, rank, world)

    cpu = cfg0 = None
    procs = host_cores()
    if world == 1 and not args.no_cfg0:
        cfg0 = configs0_inference(args, rank, procs)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, dt = cpu_baseline(ds, args.hidden, args.batch, args.cpu_steps, procs)
        cpu = {"value": v, "unit": "graphs/s", "cores": procs, "kind": "port",
               "sample": f"{args.cpu_steps} steps x {args.batch} graphs of the same corpus: oracle gnn.backward + "
                         f"Adam (fp64 numpy), {procs} procs x 1 BLAS thread, {cpu_model()}, {dt:.1f} s"}

    if rank == 0:
        step_ms = ms / args.steps
        line = {"metric": METRIC, "value": value, "unit": "graphs/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": args.dtype, "data": DATA, "config": config_dict(args, world),
                "e2e": e2e, "gpu_launches": int(launches),
                "roofline": {"bound": "tensor", "kernel": "k_tc_gemm (tcgen05 fwd/dgrad/wgrad, all launches)",
                             "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s", "frac": achieved / peak_tf,
                             "traffic": traffic,
                             "peak_source": pk_src + ": burst bf16 (each GEMM is event-timed alone in a short "
                                            "eager pass)" + ("" if args.dtype == "bf16" else
                                                             "; fp32 mode = 3-pass tf32: bf16 burst / 2 / 3"),
                             "gemm_share_of_step": (g_ms / args.steps) / step_ms,
                             "gemm_launches_per_step": g_n / args.steps,
                             "algorithmic_tflop_per_step": step_flops / 1e12,
                             "by_class": {k: dict(v, frac=(v["tflops"] or 0.0) / peak_tf)
                                          for k, v in timer.classes(args.steps).items()},
                             "whole_step": {"tflops": step_flops / (step_ms / 1000.0) / 1e12,
                                            "frac": step_flops / (step_ms / 1000.0) / 1e12 / peak_tf,
                                            "what": "algorithmic GEMM FLOPs of a step / the timed step time"},
                             "hbm_kernels": dict(hbm, peak_gbs=pk["hbm_gbs"],
                                                 note="event-timed per launch in the roofline pass (the step's "
                                                      "Python orchestration, which the hooks require: the same "
                                                      "kernels as the timed native step, except that the native "
                                                      "step forms K2's layer-1 pass inside K1); algorithmic "
                                                      "bytes per DESIGN.md §3")},
                "cpu_baseline": cpu, "clocks": clocks, "wall_s_timed_region": wall, "train_fp32": train_fp32,
                "configs0_inference": cfg0, "inference": infer}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
