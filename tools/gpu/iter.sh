# One iteration call: targeted tests, the in-stream step breakdown, the serialised launch list.
set -x
timeout 600 python -m pytest -q -x -p no:cacheprovider ${TESTS:-tests/test_gpu_kernels.py tests/test_gpu_headline.py} 2>&1 | tail -3
timeout 300 python tools/step_breakdown.py bf16 2>&1 | tail -30
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/one_step.py > /dev/null 2>&1
python tools/ncu_metrics.py gpurun_out/launches.csv
