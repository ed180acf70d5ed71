"""Data-parallel training on the device path, two ranks sharing one GPU (gloo carries the
all-reduce; the pool grants one GPU, so NCCL itself is not exercised here).

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
