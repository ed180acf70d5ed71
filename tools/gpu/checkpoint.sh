# Round checkpoint: full GPU suite, bench line, step launch list.
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/ck_bench.json 2> gpurun_out/ck_bench.err; tail -2 gpurun_out/ck_bench.err
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ck_launches.csv python tools/one_step.py > /dev/null 2>&1
python tools/ncu_metrics.py gpurun_out/ck_launches.csv > gpurun_out/ck_launches.txt; cat gpurun_out/ck_launches.txt
