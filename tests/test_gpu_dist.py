"""Data-parallel training on the device path, two ranks sharing one GPU (gloo carries the
all-reduce; the pool grants one GPU, so NCCL itself runs only as a one-rank group, in
test_nccl_one_rank_collectives_on_device).

Each rank runs the engine's forward / loss (global-batch gradient denominator) / backward
with the two-bucket OverlappedAllReduce of BatchTrainer._step on its half of a batch; the
summed gradients must equal the single-process gradients of the whole batch (same kernels,
different accumulation order across the two halves: tolerance per dtype).  bf16 runs the
fused head (deferred to the backward, the first bucket issued after the layer-3 weight
gradient), fp32 the per-op head."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _grads(prec, ids, global_g, allreduce=None):
    import torch

    from paper_2303_11733_b200 import gnn
    from paper_2303_11733_b200.device import Engine, Workspace, upload_batch
    from paper_2303_11733_b200.synth import make_dataset
    ds = make_dataset(256, seed=23)
    norm = gnn.Normalizer.fit(ds.y.astype(np.float64), ds.fs.astype(np.float64))
    model = gnn.create_model(hidden=256, seed=6, normalizer=norm)
    eng = Engine(256, prec)
    eng.set_params(model.param_items(), model.normalizer)
    b = upload_batch(*ds.collate(ids), device="cuda")
    ws = Workspace(eng, b.N, b.G, train=True)
    eng.grads.zero_()
    eng.forward(b, ws, predict=False, defer_head=True)
    eng.loss(b, ws, 1.0, grad_den=float(global_g))
    if allreduce is None:
        eng.backward(b, ws)
    else:
        split = {}

        def first_bucket(off):
            split["off"] = off
            allreduce.begin(eng.grads[off:])
        eng.backward(b, ws, on_partial=first_bucket)
        allreduce.begin(eng.grads[:split["off"]])
        allreduce.finish()
    torch.cuda.synchronize()
    return eng.get_grads()


def _worker(rank, port, prec, out):
    import torch.distributed as dist

    from paper_2303_11733_b200.dist import OverlappedAllReduce
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        ids = np.arange(rank * 128, (rank + 1) * 128)
        g = _grads(prec, ids, 256, OverlappedAllReduce())
        if rank == 0:
            np.savez(out, **g)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("prec,rel", [("fp32", 1e-4), ("bf16", 2e-2)])
def test_data_parallel_step_equals_single_process(tmp_path, prec, rel):
    import torch.multiprocessing as mp
    out = str(tmp_path / "dp.npz")
    mp.spawn(_worker, args=(_free_port(), prec, out), nprocs=2, join=True)
    dp = dict(np.load(out))
    ref = _grads(prec, np.arange(256), 256)
    for name, g in ref.items():
        err = np.linalg.norm(dp[name] - g) / max(np.linalg.norm(g), 1e-30)
        assert err < rel, (name, err)


class _ForcedAllReduce:
    """OverlappedAllReduce with the world-size gate removed, so a one-rank NCCL group still
    issues the asynchronous all-reduces (sum over one rank: the identity)."""

    def __new__(cls):
        from paper_2303_11733_b200.dist import OverlappedAllReduce

        class Forced(OverlappedAllReduce):
            def _active(self):
                return True
        return Forced()


def _nccl_worker(rank, port, out):
    import torch
    import torch.distributed as dist

    from paper_2303_11733_b200.dist import gather_predictions, global_batch_size
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        assert dist.get_backend() == "nccl"
        g = _grads("bf16", np.arange(256), 256, _ForcedAllReduce())
        assert global_batch_size(256) == 256
        y = torch.arange(12, dtype=torch.float32, device="cuda").view(4, 3)
        mig = torch.tensor([0, 1, -1, 3], dtype=torch.int8, device="cuda")
        ys, ms = gather_predictions(y, mig)
        assert torch.equal(ys, y) and torch.equal(ms, mig)
        np.savez(out, **g)
    finally:
        dist.destroy_process_group()


def test_nccl_one_rank_collectives_on_device():
    """The NCCL leg of the DP path on the one GPU the pool grants: a one-rank NCCL group runs
    the two-bucket asynchronous gradient all-reduce inside the backward (issued on NCCL's
    stream after the layer-3 weight gradient, waited on before Adam), the global-batch
    all-reduce and the prediction all-gather; the gradients are bit-identical to the
    no-collective step (a one-rank sum is the identity, and the ordering must not race)."""
    import tempfile

    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "nccl.npz")
        mp.spawn(_nccl_worker, args=(_free_port(), out), nprocs=1, join=True)
        got = dict(np.load(out))
    ref = _grads("bf16", np.arange(256), 256)
    for name, g in ref.items():
        assert np.array_equal(got[name], g), name


def _trainer_worker(rank, port, native, out):
    import copy

    import torch
    import torch.distributed as dist

    from paper_2303_11733_b200 import gnn, trainer as trainer_mod
    from paper_2303_11733_b200.device import upload_batch
    from paper_2303_11733_b200.dist import OverlappedAllReduce
    from paper_2303_11733_b200.synth import make_dataset
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        trainer_mod.NATIVE_STEP = native
        ds = make_dataset(256, seed=29)
        norm = gnn.Normalizer.fit(ds.y.astype(np.float64), ds.fs.astype(np.float64))
        model = gnn.create_model(hidden=256, seed=8, normalizer=norm)
        tr = trainer_mod.BatchTrainer(copy.deepcopy(model), precision="bf16", lr=1e-3, seed=5,
                                      allreduce=OverlappedAllReduce(), world_size=2, rank=rank)
        for k in range(2):  # rank r takes graphs [r * 64, (r + 1) * 64) of each 128-graph batch
            ids = np.arange(k * 128 + rank * 64, k * 128 + (rank + 1) * 64)
            tr.step_resident(upload_batch(*ds.collate(ids), device="cuda", build_csr=False))
        torch.cuda.synchronize()
        assert (tr._native is not None) == native
        if rank == 0:
            np.save(out, tr.engine.params.cpu().numpy())
    finally:
        dist.destroy_process_group()


def test_data_parallel_native_step_equals_python_step(tmp_path):
    """Two ranks (gloo, sharing the GPU) training through BatchTrainer with the all-reduce:
    the native executor (gradients, one all-reduce, Adam) and the Python orchestration (its
    two overlapped buckets) end with bit-identical parameters."""
    import torch.multiprocessing as mp
    res = []
    for native in (True, False):
        out = str(tmp_path / f"dp_{int(native)}.npy")
        mp.spawn(_trainer_worker, args=(_free_port(), native, out), nprocs=2, join=True)
        res.append(np.load(out))
    assert np.array_equal(res[0], res[1])
