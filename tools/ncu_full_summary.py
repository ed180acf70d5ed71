"""Key numbers of one kernel from an `ncu --set full` report: speed-of-light, memory,
occupancy, scheduler and the top warp-stall reasons (text, for profiles/)."""
import csv
import io
import subprocess
import sys

KEEP = ("Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput",
        "L1/TEX Cache Throughput", "Compute (SM) Throughput", "SM Active Cycles", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "Issued Warp Per Scheduler",
        "No Eligible", "Eligible Warps Per Scheduler", "Grid Size", "Block Size")


def main(rep):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(det)))
    h = rows[0]
    ki, mi, vi, ui = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    print(rows[1][ki][:120])
    seen = set()
    for r in rows[1:]:
        if r[mi] in KEEP and r[mi] not in seen:
            seen.add(r[mi])
            print(f"  {r[mi]:32s} {r[vi]} {r[ui]}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    stalls = []
    for n, v in zip(rr[0], rr[2]):
        if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued"):
            try:
                stalls.append((float(v), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1.0
    print("  top warp-stall reasons (share of samples):",
          ", ".join(f"{name} {100 * s / tot:.0f}%" for s, name in sorted(stalls, reverse=True)[:5]))


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        main(rep)
