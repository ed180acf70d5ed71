set -x
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "cta_pair" 2>&1 | tail -15
timeout 200 python tools/gemm_bench.py 2>&1 | tail -30
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
timeout 300 python tools/step_breakdown.py bf16 2>&1 | tail -45
