"""configs[4] end-to-end predict from graph JSON at several pipeline chunk sizes (same 8192
documents): bench.predict_from_json's measurement with docs_per_batch x batches varied."""
import sys
import types

sys.path.insert(0, ".")
import bench  # noqa: E402

args = types.SimpleNamespace(hidden=512)
for per, nb in [(4096, 2), (2048, 4), (1024, 8), (512, 16)]:
    r = bench.predict_from_json(args, 0, 1, docs_per_batch=per, batches=nb)
    print(f"chunk {per:5d} x {nb:2d}: {r['docs_per_s']:8.0f} docs/s end to end "
          f"(featurise {r['featurise_docs_per_s']:.0f}, device {r['device_docs_per_s']:.0f})", flush=True)
