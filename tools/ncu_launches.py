"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel."""
import collections
import csv
import sys


def load(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    if "Metric Name" in hdr:  # several metrics per launch: keep the duration rows
        mi = hdr.index("Metric Name")
        rows = [hdr] + [r for r in rows[1:] if r[mi] == "gpu__time_duration.sum"]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    out = []
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[r[ui]]
        out.append((r[ki], v * scale))
    return out


def main(path, width=100):
    launches = load(path)
    tot = sum(t for _, t in launches)
    agg = collections.OrderedDict()
    for name, t in launches:
        a = agg.setdefault(name[:width], [0.0, 0])
        a[0] += t
        a[1] += 1
    print(f"{len(launches)} launches, {tot:.1f} us total (cold-cache, serialised)")
    for k, (t, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"{t:10.1f} us {c:4d}x {100 * t / tot:5.1f}%  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
