timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "passed|failed|^FAILED|^E  " | head -8
python tools/gemm_sweep.py 2
timeout 600 python bench.py --no-cpu-baseline --no-infer --no-e2e 2>&1 | tail -1 | cut -c 1-250
