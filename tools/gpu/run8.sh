timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -2
timeout 200 python tools/gemm_bench.py 2>&1 | grep "pair2\|l1"
timeout 200 python tools/gemm_sweep.py 2>&1 | head -2
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1s2_step_ncu8.csv python tools/one_step.py > /dev/null 2>&1
python tools/ncu_list.py gpurun_out/r1s2_step_ncu8.csv | grep tc_gemm | cut -c 1-110
timeout 500 python bench.py --no-cpu-baseline --no-infer 2>&1 | tail -1 | cut -c 1-300
