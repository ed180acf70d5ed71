"""Does in-process NVML sampling perturb a running CUDA workload? (bench clocks design)"""
import threading
import time
import sys

import pynvml
import torch

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)


def run(n=200):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        a @ a
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e3


stop = False
samples = []


def sampler(ms, reasons):
    while not stop:
        c = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h) if reasons else 0
        samples.append((c, r))
        time.sleep(ms / 1000)


run(20)
print("baseline ms/gemm", run())
for ms, reasons in ((200, False), (200, True), (50, True)):
    stop = False
    samples.clear()
    th = threading.Thread(target=sampler, args=(ms, reasons))
    th.start()
    v = run()
    stop = True
    th.join()
    print(f"nvml every {ms} ms reasons={reasons}: ms/gemm {v:.3f}, {len(samples)} samples, last {samples[-1]}")
