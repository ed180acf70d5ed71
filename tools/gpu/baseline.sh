set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 300 python tools/step_breakdown.py bf16 2>&1 | tail -30
timeout 900 python bench.py > gpurun_out/base_bench.json 2> gpurun_out/base_bench.err; tail -3 gpurun_out/base_bench.err
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/one_step.py > /dev/null 2>&1
python tools/ncu_metrics.py gpurun_out/launches.csv
