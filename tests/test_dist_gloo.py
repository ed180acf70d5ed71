"""Multi-process (world size 2, gloo, CPU) tests of the data-parallel and
sharded-inference logic in paper_2303_11733_b200/dist.py.

The GPU kernels are exercised by the -m gpu suite; here the per-rank compute is
the CPU oracle, so what is tested is exactly the host-side N>1 logic:
sharding by node count, the global-batch gradient denominator + the two-bucket
SUM all-reduce reproducing the single-process gnn.backward mean (gnn.py:402-404),
and the ordered all-gather of per-rank predictions."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import unpack_records
from oracle import dippm_oracle as O
from paper_2303_11733_b200.dist import OverlappedAllReduce, gather_predictions, global_batch_size, shard_by_nodes

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _params_norm(golden):
    params = O.init_params(32, np.random.default_rng(11))
    for k in O.SAGE_PARAM_NAMES:
        if params[k].ndim == 1:
            params[k] = golden[f"h32_bias_{k}"].copy()
    norm = {"y_mean": golden["norm_y_mean"], "y_std": golden["norm_y_std"],
            "fs_mean": golden["norm_fs_mean"], "fs_std": golden["norm_fs_std"]}
    return params, norm


def _worker(rank, port, golden, out):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        recs = unpack_records(golden)[:34]
        params, norm = _params_norm(golden)
        shards = shard_by_nodes([r[0] for r in recs], WORLD)
        lo, hi = shards[rank]
        mine = recs[lo:hi]
        g_total = global_batch_size(len(mine))
        # per-rank gradient share with the GLOBAL denominator (what the Huber kernel's grad_den does)
        loss, grads = O.backward(params, norm, mine)
        share = len(mine) / g_total
        flat = torch.from_numpy(np.concatenate([grads[k].ravel() * share for k in O.SAGE_PARAM_NAMES]))
        # the trainer's two buckets: head + sage3 first (overlapping the backward), then the rest
        off = sum(grads[k].size for k in O.SAGE_PARAM_NAMES[:O.SAGE_PARAM_NAMES.index("sage3.w_self")])
        ar = OverlappedAllReduce()
        ar.begin(flat[off:])
        ar.begin(flat[:off])
        ar.finish()
        # sharded inference + ordered gather
        y = torch.from_numpy(np.stack([O.predict(params, norm, *r[:4]) for r in mine]))
        mig = torch.tensor([O.mig_code(float(v)) for v in y[:, 1]], dtype=torch.int8)
        ys, ms = gather_predictions(y, mig)
        if rank == 0:
            out.put((g_total, flat.numpy(), ys.numpy(), ms.numpy(), shards))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_data_parallel_gradients_and_sharded_inference(golden):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, golden, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    g_total, flat, ys, ms, shards = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    recs = unpack_records(golden)[:34]
    params, norm = _params_norm(golden)
    assert g_total == len(recs)
    _, ref = O.backward(params, norm, recs)
    ref_flat = np.concatenate([ref[k].ravel() for k in O.SAGE_PARAM_NAMES])
    assert np.allclose(flat, ref_flat, rtol=1e-12, atol=1e-15)
    ref_y = np.stack([O.predict(params, norm, *r[:4]) for r in recs])
    assert np.array_equal(ys, ref_y)
    assert ms.tolist() == [O.mig_code(float(v)) for v in ref_y[:, 1]]
    assert shards[0][0] == 0 and shards[-1][1] == len(recs)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_by_nodes_balanced_and_complete(world):
    rng = np.random.default_rng(world)
    n = np.concatenate([rng.integers(270, 331, 500), rng.integers(2, 5000, 40)])
    rng.shuffle(n)
    shards = shard_by_nodes(n, world)
    assert len(shards) == world
    assert shards[0][0] == 0 and shards[-1][1] == len(n)
    assert all(a[1] == b[0] for a, b in zip(shards, shards[1:]))
    loads = [n[a:b].sum() for a, b in shards]
    assert max(loads) - min(loads) <= 2 * n.max()
