"""In-stream time of every C-ABI call of a training step (CUDA events around
each call on the launching stream; real overlap/launch behaviour, unlike the
serialised ncu launch list)."""
import collections
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2303_11733_b200 import _lib, gnn  # noqa: E402
from paper_2303_11733_b200.device import upload_batch  # noqa: E402
from paper_2303_11733_b200.synth import make_dataset  # noqa: E402
from paper_2303_11733_b200.trainer import BatchTrainer  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
ds = make_dataset(2560, seed=2)
perm = np.random.default_rng(7).permutation(ds.num_graphs)
res = [upload_batch(*ds.collate(perm[i * 256:(i + 1) * 256]), build_csr=False) for i in range(10)]
model = gnn.create_model(hidden=512, seed=0, normalizer=gnn.Normalizer.fit(ds.y.astype(float), ds.fs.astype(float)))
tr = BatchTrainer(model, precision=prec)
tr.reserve(max(b.N for b in res), 256)
for i in range(5):
    tr.step_resident(res[i])
torch.cuda.synchronize()

records = []
orig_call = _lib.call
orig_check = _lib.check


def timed_call(name, *args):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    orig_call(name, *args)
    e1.record()
    records.append((name, e0, e1))


gemm_kind = {0: "gemm_fwd", 1: "gemm_store", 2: "gemm_wgrad", 3: "gemm_gate"}
lib = _lib.load()
orig_gemm = lib.dippm_gemm


class GemmWrap:
    def __call__(self, args, backend, stream):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = orig_gemm(args, backend, stream)
        e1.record()
        m = "G" if args.M <= 8192 and args.kind != 2 else ("N" if args.kind != 2 else "H")
        records.append((f"{gemm_kind[args.kind]} M={m} N{args.N} K{'rows' if args.K > 8192 else args.K}", e0, e1))
        return r


_lib.call = timed_call
lib.dippm_gemm = GemmWrap()
steps = 5
torch.cuda.synchronize()
t0 = torch.cuda.Event(enable_timing=True)
t1 = torch.cuda.Event(enable_timing=True)
t0.record()
for i in range(steps):
    tr.step_resident(res[5 + i])
t1.record()
torch.cuda.synchronize()
total = t0.elapsed_time(t1) / steps
agg = collections.OrderedDict()
for name, a, b in records:
    v = agg.setdefault(name, [0.0, 0])
    v[0] += a.elapsed_time(b) / steps
    v[1] += 1
print(f"{prec}: {total * 1e3:.1f} us per step (with event overhead); per call (us/step):")
acc = 0.0
for name, (t, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    acc += t
    print(f"{t * 1e3:8.1f}  x{c // steps:<3d} {name}")
print(f"sum {acc * 1e3:.1f} us")
