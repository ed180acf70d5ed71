"""Per-call device time of the C-ABI kernels of one bf16 training step, each call re-run in
isolation (CUDA events around `reps` back-to-back launches on the launching stream, after a
warm-up).  The GEMMs (dippm_gemm) are skipped: tools/gemm_probe.py covers them.
usage: python tools/call_bench.py [regex] [reps]"""
import re
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2303_11733_b200 import _lib, gnn  # noqa: E402
from paper_2303_11733_b200.device import upload_batch  # noqa: E402
from paper_2303_11733_b200.synth import make_dataset  # noqa: E402
from paper_2303_11733_b200.trainer import BatchTrainer  # noqa: E402

pat = re.compile(sys.argv[1] if len(sys.argv) > 1 else ".")
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
ds = make_dataset(1536, seed=2)
perm = np.random.default_rng(7).permutation(ds.num_graphs)
res = [upload_batch(*ds.collate(perm[i * 256:(i + 1) * 256]), build_csr=False) for i in range(6)]
model = gnn.create_model(hidden=512, seed=0, normalizer=gnn.Normalizer.fit(ds.y.astype(float), ds.fs.astype(float)))
tr = BatchTrainer(model, precision="bf16")
tr.reserve(max(b.N for b in res), 256)
for i in range(4):
    tr.step_resident(res[i])
torch.cuda.synchronize()
calls = []
orig = _lib.call


def rec(name, *args):
    calls.append((name, args, torch.cuda.current_stream()))
    orig(name, *args)


_lib.call = rec
tr.step_resident(res[4])
torch.cuda.synchronize()
_lib.call = orig
print(f"N = {res[4].N} nodes, G = {res[4].G}")
seen = {}
for name, args, stream in calls:
    if not pat.search(name):
        continue
    k = seen.get(name, 0)
    seen[name] = k + 1
    with torch.cuda.stream(stream):
        for _ in range(3):
            orig(name, *args)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            orig(name, *args)
        e1.record()
    torch.cuda.synchronize()
    print(f"{e0.elapsed_time(e1) / reps * 1e3:8.1f} us  {name}#{k}")
