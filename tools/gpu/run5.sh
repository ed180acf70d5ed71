timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1s2_step_ncu5.csv python tools/one_step.py > /dev/null 2>&1
python tools/ncu_launches.py gpurun_out/r1s2_step_ncu5.csv | head -40
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_adam_pack -c 1 -o gpurun_out/r1s2_adam_full python tools/one_step.py > /dev/null 2>&1
timeout 500 python bench.py --no-cpu-baseline --no-infer 2>&1 | tail -1 | cut -c 1-300
