timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "wgrad" 2>&1 | tail -2
timeout 200 python tools/gemm_bench.py 2>&1 | grep bf16
timeout 300 python tools/step_breakdown.py bf16 2>&1 | tail -30
timeout 500 python bench.py --no-cpu-baseline --no-infer 2>&1 | tail -1 | cut -c 1-400
