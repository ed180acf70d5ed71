"""Summarise an `ncu --set full` report of the step's tcgen05 GEMM launches: per-launch time,
DRAM bytes, tensor-pipe activity; writes the average DRAM bytes per launch (the bench's
`roofline.traffic`) to the JSON path given as the second argument."""
import csv
import io
import json
import subprocess
import sys

rep, out_json = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
unit_row = rows[1]


def col(name):
    return h.index(name) if name in h else None


ki = col("Kernel Name")
ti, dr, dw = col("gpu__time_duration.sum"), col("dram__bytes_read.sum"), col("dram__bytes_write.sum")
tp = col("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed") or col(
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}
tot_b, n = 0.0, 0
print("kernel | time_us | dram_read_MB | dram_write_MB | tensor_pipe_active_pct")
for r in rows[2:]:
    if not r or "k_tc_gemm" not in r[ki]:
        continue
    t = float(r[ti].replace(",", "")) * scale.get(unit_row[ti], 1)
    rb = float(r[dr].replace(",", "")) * scale.get(unit_row[dr], 1)
    wb = float(r[dw].replace(",", "")) * scale.get(unit_row[dw], 1)
    tpv = r[tp] if tp is not None else "n/a"
    name = r[ki].split("(")[0].replace("void ", "").replace("dippm::tc::", "")
    print(f"{name} | {t:.1f} | {rb / 1e6:.1f} | {wb / 1e6:.1f} | {tpv}")
    tot_b += rb + wb
    n += 1
summary = {"source": f"{rep} (ncu --set full, one training step's {n} k_tc_gemm launches, bf16)",
           "gemm_dram_bytes_per_launch_bf16": tot_b / max(n, 1), "gemm_launches": n}
json.dump(summary, open(out_json, "w"), indent=1)
print(json.dumps(summary))
