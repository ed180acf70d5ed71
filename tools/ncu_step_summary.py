"""Per-kernel key numbers of an `ncu --set full` capture of one training step (every launch):
duration, DRAM bytes (read + write) and throughput, L2 throughput, tensor-pipe activity,
achieved occupancy, registers, and the top warp-stall reasons.  Writes the GEMM launches'
mean DRAM bytes to the JSON given as the second argument (the bench's roofline.traffic).
usage: python tools/ncu_step_summary.py REPORT.ncu-rep [ncu_summary.json]"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]


units = rows[1]
SCALE = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def get(r, name, scale=1.0):
    """Metric value in base units (seconds, bytes) times scale; percentages as given."""
    if name not in h:
        return None
    i = h.index(name)
    try:
        v = float(r[i].replace(",", ""))
    except ValueError:
        return None
    return v * SCALE.get(units[i], 1.0) * scale


print(f"{'kernel':44s} {'us':>7s} {'DRAM MB':>8s} {'DRAM%':>6s} {'L2%':>5s} {'tensor%':>7s} {'occ%':>5s} {'regs':>4s}  top stalls")
gemm_bytes = []
for r in rows[2:]:
    name = r[h.index("Kernel Name")]
    us = get(r, "gpu__time_duration.sum", 1e6)
    rd, wr = get(r, "dram__bytes_read.sum") or 0.0, get(r, "dram__bytes_write.sum") or 0.0
    dram = get(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")
    l2 = get(r, "lts__throughput.avg.pct_of_peak_sustained_elapsed")
    tens = get(r, "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active")
    if tens is None:
        tens = get(r, "sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active")
    occ = get(r, "sm__warps_active.avg.pct_of_peak_sustained_active")
    regs = get(r, "launch__registers_per_thread")
    stalls = []
    for i, n in enumerate(h):
        if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued"):
            try:
                stalls.append((float(r[i].replace(",", "")), n[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(v for v, _ in stalls) or 1.0
    top = ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in sorted(stalls, reverse=True)[:3])
    short = name.replace("void ", "").replace("tc::", "").split("(")[0][:44]
    if "k_tc_gemm" in name:
        gemm_bytes.append(rd + wr)
    f = lambda x, fmt: (fmt % x) if x is not None else "-"
    print(f"{short:44s} {f(us, '%7.1f')} {(rd + wr) / 1e6:8.1f} {f(dram, '%6.1f')} {f(l2, '%5.1f')} {f(tens, '%7.1f')} "
          f"{f(occ, '%5.1f')} {f(regs, '%4.0f')}  {top}")
if len(sys.argv) > 2 and gemm_bytes:
    json.dump({"source": f"{rep} (ncu --set full, one training step, bf16)",
               "gemm_dram_bytes_per_launch_bf16": sum(gemm_bytes) / len(gemm_bytes), "gemm_launches": len(gemm_bytes)},
              open(sys.argv[2], "w"), indent=1)
