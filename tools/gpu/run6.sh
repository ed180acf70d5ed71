timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -2
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1s2_step_ncu6.csv python tools/one_step.py > /dev/null 2>&1
python tools/ncu_list.py gpurun_out/r1s2_step_ncu6.csv | cut -c 1-120
timeout 500 python bench.py --no-cpu-baseline --no-infer 2>&1 | tail -1 | cut -c 1-300
