"""Golden fixtures for the native featuriser (§8f row 1), produced by the REAL
reference in the build container:

    python tests/golden/make_golden_featurize.py

For each graph JSON document it records what the reference's front end
returns — parse_graph_json [graph_ir.py:212-297] (re-topologise, validate,
infer_shapes [:357-499]), optional with_batch_size [:502-529], then
create_graph_encoding [featurize.py:186-190] and static_features [:256-267] —
or the name of the DippmError subclass it raises.  Documents: zoo models of
every family [graph_ir.py:577], random_graph [tests/helpers.py:55] (whole
vocabulary, consts, bmm detours, skips), non-canonical rewrites (shuffled ids,
missing shapes, float attrs, namespaced / cased op names, unknown keys) and
malformed documents for every error path.
"""

from __future__ import annotations

import json
import random
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

from dippm import featurize, graph_ir  # noqa: E402
from dippm.errors import DippmError  # noqa: E402
from helpers import random_graph  # noqa: E402

OUT = Path(__file__).resolve().parent / "golden_featurize_v1.npz"


def zoo_docs():
    specs = [("resnetish", 60, 8, 2, 16, 7), ("mlp", 150, 8, 1, 8, 1), ("vggish", 3, 4, 4, 32, 2),
             ("resnetish", 3, 4, 1, 8, 11), ("vggish", 1, 2, 2, 8, 5), ("mlp", 2, 16, 8, 16, 3),
             ("resnetish", 12, 8, 4, 32, 21), ("vggish", 5, 8, 1, 64, 9)]
    return [graph_ir.serialize_graph(graph_ir.build_zoo_model(graph_ir.ZooSpec(*s))) for s in specs]


def rewrite(doc_text, rng, shuffle=True, drop_shapes=False, float_attrs=False, rename=False, extra=False):
    doc = json.loads(doc_text)
    nodes = doc["nodes"]
    ids = list(range(len(nodes)))
    new_id = ids[:]
    if shuffle:
        new_id = list(rng.permutation(len(nodes)) * 3 + 5)
    for nd in nodes:
        nd["id"] = int(new_id[nd["id"]])
        nd["inputs"] = [int(new_id[i]) for i in nd["inputs"]]
        if drop_shapes and nd["inputs"] and "out_shape" in nd and nd["op"] not in ("reshape",):
            del nd["out_shape"]
        if float_attrs:
            nd["attrs"] = {k: float(v) for k, v in nd["attrs"].items()}
        if rename:
            nd["op"] = rng.choice(["nn.", "Relay.", "", "  "]) + (nd["op"].upper() if rng.random() < 0.5 else nd["op"])
        if extra:
            nd["comment"] = "x"
    doc["outputs"] = [int(new_id[o]) for o in doc["outputs"]]
    if shuffle:
        rng.shuffle(nodes)
    if extra:
        doc["producer"] = {"tool": "test", "v": [1, 2.5, None, True]}
    return json.dumps(doc, indent=1 if extra else None)


def error_docs():
    ok = {"name": "e", "batch": 1, "outputs": [1],
          "nodes": [{"id": 0, "op": "input", "inputs": [], "attrs": {}, "out_shape": [1, 4]},
                    {"id": 1, "op": "dense", "inputs": [0], "attrs": {"out_features": 3}}]}

    def mod(f):
        d = json.loads(json.dumps(ok))
        f(d)
        return json.dumps(d)

    docs = ["{not json", "[1, 2]", json.dumps({"batch": 1, "outputs": [0], "nodes": []}),
            mod(lambda d: d.update(outputs=[])), mod(lambda d: d.update(outputs=[1.0])),
            mod(lambda d: d.update(batch=0)), mod(lambda d: d.update(batch=1.5)), mod(lambda d: d.update(batch=True)),
            mod(lambda d: d.update(name=3)), mod(lambda d: d["nodes"][1].update(id=0)),
            mod(lambda d: d["nodes"][1].update(id=-1)), mod(lambda d: d["nodes"][1].update(op="")),
            mod(lambda d: d["nodes"][1].update(inputs=[0.0])), mod(lambda d: d["nodes"][1].update(attrs={"a": True})),
            mod(lambda d: d["nodes"][0].update(out_shape=[1, 2, 3, 4, 5])),
            mod(lambda d: d["nodes"][0].update(out_shape=[1, 0])), mod(lambda d: d["nodes"][0].update(out_shape=[1, 2.0])),
            mod(lambda d: d["nodes"][0].update(out_shape=None)), mod(lambda d: d["nodes"][1].update(inputs=[7])),
            mod(lambda d: d.update(outputs=[9])), mod(lambda d: d["nodes"][0].update(inputs=[1])),
            mod(lambda d: d["nodes"][1].update(op="const")),
            mod(lambda d: d["nodes"][1].update(op="conv2d")),
            mod(lambda d: d["nodes"][1].update(op="conv2d", attrs={"kernel_h": 1, "kernel_w": 1, "out_features": 2})),
            mod(lambda d: d["nodes"][1].update(op="batch_matmul")),
            mod(lambda d: d["nodes"][1].update(attrs={})), mod(lambda d: d["nodes"][0].update(out_shape="x")),
            mod(lambda d: d["nodes"].append("x")), mod(lambda d: d["nodes"][1].update(inputs=5)),
            mod(lambda d: d["nodes"][1].update(attrs=[1])),
            ]
    return docs


def run(text, batch):
    try:
        g = graph_ir.parse_graph_json(text)
        if batch:
            g = graph_ir.with_batch_size(g, batch)
        enc = featurize.create_graph_encoding(g)
        fs = featurize.static_features(g)
        return None, g.name, enc, fs
    except DippmError as exc:
        return type(exc).__name__, None, None, None


def main():
    rng = np.random.default_rng(17)
    prng = random.Random(99)
    docs = []  # (text, batch override)
    for d in zoo_docs():
        docs.append((d, 0))
    for i in range(40):
        docs.append((graph_ir.serialize_graph(random_graph(prng, small=(i % 4 == 0))), 0))
    base = [d for d, _ in docs]
    for i, d in enumerate(base[:20]):
        docs.append((rewrite(d, rng, shuffle=True, drop_shapes=(i % 2 == 0), float_attrs=(i % 3 == 0),
                             rename=(i % 4 == 1), extra=(i % 5 == 2)), 0))
    for i, d in enumerate(base[:10]):
        docs.append((d, [1, 3, 8, 16, 2][i % 5]))
    for d in error_docs():
        docs.append((d, 0))
    docs.append((base[0], -1))  # with_batch_size(-1) -> InvalidSpec

    errors, names, n, ne, edges, x, fs = [], [], [], [], [], [], []
    for text, b in docs:
        err, name, enc, st = run(text, b)
        errors.append(err or "")
        names.append(name or "")
        if err:
            n.append(0)
            ne.append(0)
            fs.append([0] * 5)
            continue
        n.append(enc.num_nodes)
        ne.append(len(enc.edges))
        edges.extend(enc.edges)
        x.append(enc.features)
        fs.append([st.macs, st.batch, st.t_conv, st.t_dense, st.t_relu])
    blob = [t.encode("utf-8") for t, _ in docs]
    offs = np.zeros(len(blob) + 1, np.int64)
    np.cumsum([len(b) for b in blob], out=offs[1:])
    out = {
        "doc_bytes": np.frombuffer(b"".join(blob), dtype=np.uint8), "doc_offsets": offs,
        "batch_override": np.array([b for _, b in docs], np.int64),
        "error": np.array(errors), "name": np.array(names),
        "n": np.array(n, np.int64), "ne": np.array(ne, np.int64),
        "edges": np.array(edges, np.int64).reshape(-1, 2), "x": np.concatenate(x),
        "fs_int": np.array(fs, np.int64),
    }
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1024:.1f} KiB): {len(docs)} docs, "
          f"{sum(1 for e in errors if e)} errors, {sum(n)} nodes; error kinds {sorted(set(e for e in errors if e))}")


if __name__ == "__main__":
    main()
