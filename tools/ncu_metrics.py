"""Per-kernel time + DRAM bytes from `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,...--csv`."""
import collections
import csv
import sys

TIME = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
BYTES = {"byte": 1, "B": 1, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9}


def load(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    h = rows[0]
    ki, mi, vi, ui, ii = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    per = collections.OrderedDict()
    for r in rows[1:]:
        d = per.setdefault(r[ii], {"name": r[ki]})
        v = float(r[vi].replace(",", ""))
        d[r[mi]] = v * (TIME.get(r[ui]) or BYTES.get(r[ui]) or 1.0)
    return list(per.values())


def main(path):
    per = load(path)
    tot = sum(d["gpu__time_duration.sum"] for d in per)
    print(f"{len(per)} launches, {tot:.1f} us (ncu: cold cache, serialised)")
    agg = collections.OrderedDict()
    for d in per:
        a = agg.setdefault(d["name"][:80], [0.0, 0, 0.0])
        a[0] += d["gpu__time_duration.sum"]
        a[1] += 1
        a[2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    for n, (t, c, b) in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"{t:8.1f} us {c:3d}x {100 * t / tot:5.1f}%  dram {b / 1e6:8.1f} MB {b / t / 1e3:6.0f} GB/s  {n}")


if __name__ == "__main__":
    main(sys.argv[1])
