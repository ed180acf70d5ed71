"""Device (fp32 = 3-pass tf32) loss / gradient error against the fp64 oracle across hidden
widths, beside the oracle's own sensitivity: its gradients under a 1e-5 relative perturbation of
the weights (ReLU units near zero flip).  Usage: python tools/width_errors.py [hidden ...]
(the device leg needs a GPU; --oracle-only runs the sensitivity leg alone on CPU)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import dippm_oracle as O  # noqa: E402
from paper_2303_11733_b200 import gnn  # noqa: E402
from paper_2303_11733_b200.device import Layout  # noqa: E402
from paper_2303_11733_b200.synth import make_dataset  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
oracle_only = "--oracle-only" in sys.argv


def nrel(a, r):
    return np.linalg.norm(a - r) / (np.linalg.norm(r) + 1e-300)


for hidden in [int(h) for h in (args or [150, 300, 512, 700, 1000])]:
    ds = make_dataset(12, seed=hidden, n_lo=20, n_hi=80)
    norm = gnn.Normalizer.fit(ds.y.astype(np.float64), ds.fs.astype(np.float64))
    model = gnn.create_model(hidden=hidden, seed=4, normalizer=norm)
    batch = ds.records(range(12))
    params = {k: np.array(v) for k, v in model.param_items()}
    nd = {"y_mean": norm.y_mean, "y_std": norm.y_std, "fs_mean": norm.fs_mean, "fs_std": norm.fs_std}
    orecs = [(r.encoding.num_nodes, r.encoding.edges, r.encoding.features, r.fs.as_vector, r.target.as_array)
             for r in batch]
    ref_loss, ref = O.backward(params, nd, orecs)
    rng = np.random.default_rng(0)
    _, pert = O.backward({k: v * (1 + 1e-5 * rng.standard_normal(v.shape)) for k, v in params.items()}, nd, orecs)
    print(f"hidden {hidden} (hp {Layout(hidden).hp})", flush=True)
    grads = None
    if not oracle_only:
        loss, grads = gnn.backward(model, batch)
        print(f"  loss rel err {abs(loss - ref_loss) / abs(ref_loss):.2e}")
    for k in O.SAGE_PARAM_NAMES:
        dev = f"device |d|/|g| {nrel(grads[k], ref[k]):.2e}   " if grads is not None else ""
        print(f"  {k:14s} {dev}oracle at 1e-5 weight perturbation {nrel(pert[k], ref[k]):.2e}", flush=True)
