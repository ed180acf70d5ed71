timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_head_fused.py tests/test_gpu_headline.py tests/test_gpu_step_native.py tests/test_gpu_model.py tests/test_gpu_kernels.py tests/test_gpu_mlp.py 2>&1 | tail -3
timeout 300 python tools/call_bench.py head 2>&1 | tail -1
