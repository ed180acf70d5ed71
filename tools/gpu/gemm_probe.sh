timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_kernels.py -k "pool or readout or fused" 2>&1 | tail -2
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_headline.py tests/test_gpu_step_native.py tests/test_gpu_scale.py 2>&1 | tail -2
for k in fwd pool; do timeout 300 python tools/gemm_probe.py $k 2>&1 | grep "K=1024" | head -2; done
bash tools/gpu/quick.sh
