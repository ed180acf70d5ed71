"""Hot SASS lines of one kernel from `ncu -i rep --page source --csv --print-source sass`:
stall-reason totals and the instructions with the most warp-stall samples."""
import csv
import sys


def main(path, n=30):
    rows = list(csv.reader(open(path)))
    h = None
    data = []
    for r in rows:
        if r and r[0] == "Address":
            h = r
            continue
        if h and len(r) == len(h):
            data.append(r)
    idx = {k: i for i, k in enumerate(h)}

    def num(r, k):
        try:
            return float(r[idx[k]] or 0)
        except ValueError:
            return 0.0

    S, I = "Warp Stall Sampling (All Samples)", "Instructions Executed"
    print(f"samples {sum(num(r, S) for r in data):.0f}  warp-instructions {sum(num(r, I) for r in data):.0f}")
    sc = [k for k in h if k.startswith("stall_")]
    tot = {k: sum(num(r, k) for r in data) for k in sc}
    s = sum(tot.values()) or 1
    print("stalls:", ", ".join(f"{k[6:]} {v / s:.0%}" for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]))
    for r in sorted(data, key=lambda r: -num(r, S))[:n]:
        top = max(sc, key=lambda k: num(r, k))
        print(f"{r[idx['Address']]:>6} {num(r, S):7.0f} {num(r, I):9.0f}  {top[6:]:<16} {r[idx['Source']][:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
