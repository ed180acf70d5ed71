python tools/wgrad_probe.py
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_kernels.py tests/test_gpu_headline.py 2>&1 | tail -2
