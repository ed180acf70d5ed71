"""Per-launch list (in launch order) from an ncu --csv metrics log."""
import sys

sys.path.insert(0, "tools")
from ncu_metrics import load  # noqa: E402

for i, d in enumerate(load(sys.argv[1])):
    t = d.get("gpu__time_duration.sum", 0)
    mb = (d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)) / 1e6
    extra = " ".join(f"{k.split('__')[-1]}={v:g}" for k, v in d.items()
                     if k not in ("name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"))
    print(f"{i:3d} {t:8.1f} us {mb:8.1f} MB  {extra}  {d['name'][:70]}")
