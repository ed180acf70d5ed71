"""Golden fixtures for the §8f "next" rows, produced by the REAL reference `dippm`.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden_next.py

Inputs are the records already pinned in golden_v1.npz (rebuilt into reference
objects), so both fixture files describe the same graphs.  Writes
tests/golden/golden_next_v1.npz with (reference file:line in brackets):
  * MLP baseline: create_mlp_model [gnn.py:307] hidden 32 / 512, forward and
    predict per record [gnn.py:348-361], backward + batch_loss over a batch
    [gnn.py:368-405], a reference-protocol train_mlp run [gnn.py:418-482]
  * dataset.mape over predictions [dataset.py:229-248]
  * JSONL lines of records [dataset.py:255-281] (interchange format the binary
    dataset sidecar converts from)
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from dippm import dataset, gnn  # noqa: E402
from dippm.dataset import DatasetRecord, TargetVector  # noqa: E402
from dippm.featurize import GraphEncoding, StaticFeatures  # noqa: E402

HERE = Path(__file__).resolve().parent
OUT = HERE / "golden_next_v1.npz"


def records_from(g, prefix):
    n, ne, edges, x, fsi, y = (g[prefix + k] for k in ("n", "ne", "edges", "x", "fs_int", "y"))
    recs, xo, eo = [], 0, 0
    for i in range(len(n)):
        enc = GraphEncoding(int(n[i]), [(int(a), int(b)) for a, b in edges[eo:eo + ne[i]]], x[xo:xo + n[i]])
        fs = StaticFeatures(*[int(v) for v in fsi[i]])
        recs.append(DatasetRecord(enc, fs, TargetVector(*[float(v) for v in y[i]]), model_name=f"rec-{i}"))
        xo += n[i]
        eo += ne[i]
    return recs


def main():
    g = dict(np.load(HERE / "golden_v1.npz"))
    recs = records_from(g, "rec_")
    norm = gnn.Normalizer(g["norm_y_mean"], g["norm_y_std"], g["norm_fs_mean"], g["norm_fs_std"])
    out = {}
    for tag, hidden, seed in (("mlp32", 32, 11), ("mlp512", 512, 0)):
        model = gnn.create_mlp_model(hidden=hidden, seed=seed, normalizer=norm)
        out[f"{tag}_param_checksum"] = np.array([float(np.sum(a)) for _, a in model.param_items()])
        brng = np.random.default_rng(seed + 200)
        for name, arr in model.param_items():
            if arr.ndim == 1:
                arr[...] = brng.normal(0.0, 0.1, size=arr.shape)
        for name, arr in model.param_items():
            if arr.ndim == 1:  # weights are rebuilt from the seed by the tests (pins the init order too)
                out[f"{tag}_bias_{name}"] = arr.copy()
        out[f"{tag}_forward"] = np.stack([gnn.forward(r.encoding, r.fs, model) for r in recs])
        out[f"{tag}_predict"] = np.stack([gnn.predict(model, r.encoding, r.fs).as_array for r in recs])
        batch = recs[:20]
        loss, grads = gnn.backward(model, batch)
        out[f"{tag}_backward_loss"] = np.array(loss)
        out[f"{tag}_batch_loss"] = np.array(gnn.batch_loss(model, batch))
        for name, gr in grads.items():
            if hidden <= 32:
                out[f"{tag}_grad_{name}"] = gr
            else:  # 512-wide gradients: per-tensor norm, sum and a strided sample
                out[f"{tag}_gradstat_{name}"] = np.array([np.linalg.norm(gr), gr.sum()])
                out[f"{tag}_gradsample_{name}"] = gr.ravel()[::97].copy()
        if tag == "mlp32":
            preds = [gnn.predict(model, r.encoding, r.fs) for r in recs]
            m = dataset.mape(preds, [r.target for r in recs])
            out["mape_mlp32"] = np.array([m.latency, m.memory, m.energy, m.overall])

    tr = records_from(g, "train_rec_")
    model, hist = gnn.train_mlp(tr[:8], tr[8:], gnn.TrainConfig(epochs=3, hidden=16, seed=123))
    out["train_mlp_hist"] = np.array([[h["epoch"], h["train_loss"], h["train_mape"], h["val_loss"], h["val_mape"]]
                                      for h in hist])
    for name, arr in model.param_items():
        out[f"train_mlp_param_{name}"] = arr.copy()

    lines = "\n".join(dataset.record_to_line(r) for r in recs[:12]) + "\n"
    out["jsonl_bytes"] = np.frombuffer(lines.encode("utf-8"), dtype=np.uint8)
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1024:.1f} KiB, {len(out)} arrays)")


if __name__ == "__main__":
    main()
