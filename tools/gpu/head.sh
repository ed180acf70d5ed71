timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_head_tc.py tests/test_gpu_head_fused.py tests/test_gpu_headline.py tests/test_gpu_step_native.py tests/test_gpu_model.py 2>&1 | tail -5
timeout 300 python tools/call_bench.py head 2>&1 | tail -1
DIPPM_HEAD_TC=0 timeout 300 python tools/call_bench.py head 2>&1 | tail -1
bash tools/gpu/quick.sh
