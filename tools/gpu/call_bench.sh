timeout 300 python tools/call_bench.py "${1:-.}" 2>&1 | tail -12
timeout 300 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_headline.py tests/test_gpu_numerics.py tests/test_gpu_step_native.py 2>&1 | tail -2
