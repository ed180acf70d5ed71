timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "passed|failed|^FAILED|^E  " | head -8
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1s2_step_ncu15.csv python tools/one_step.py > /dev/null 2>&1
python tools/ncu_list.py gpurun_out/r1s2_step_ncu15.csv | grep -v tc_gemm | cut -c 1-110
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-infer 2>&1 | tail -1 | cut -c 1-220
