"""bench.py's launch contract: `--gpus N` without torchrun spawns N ranks itself
(torch.distributed.run on 127.0.0.1) and rank 0 alone prints the JSON line.

CPU: the reference arm (the CPU oracle port) through the spawned 2-rank launch.
GPU: our arm with 2 gloo ranks sharing the one GPU of this pool (data-parallel steps with
the real all-reduce), reporting n_gpus 2 / dp2.
"""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _run(args, timeout):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd="/tmp")
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]  # rank 0 alone prints
    return json.loads(lines[0])


@pytest.mark.timeout(600)
def test_reference_arm_spawns_two_ranks_without_torchrun():
    line = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--graphs", "64",
                 "--batch", "8", "--hidden", "32"], 500)
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["config"]["parallelism"] == "dp2"
    assert line["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
@pytest.mark.timeout(900)
def test_our_arm_two_gloo_ranks_on_one_gpu():
    line = _run(["--gpus", "2", "--dist-backend", "gloo", "--steps", "3", "--warmup", "3", "--graphs", "1100",
                 "--no-infer", "--no-cpu-baseline", "--no-cfg0", "--no-fp32", "--no-clocks"], 800)
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "dp2"
    assert line["config"]["global_batch"] == 512
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
