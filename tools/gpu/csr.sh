python tools/csr_repro_tmp.py 2>&1 | tail -3
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_scale.py tests/test_gpu_kernels.py 2>&1 | tail -2
