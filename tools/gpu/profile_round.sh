# One call: tests, the bench line, the step launch list, the full GEMM capture + summary.
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/prof_bench.json 2> gpurun_out/prof_bench.err
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/prof_launches.csv python tools/one_step.py > /dev/null 2>&1
python tools/ncu_metrics.py gpurun_out/prof_launches.csv > gpurun_out/prof_launches.txt
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_tc_gemm -o gpurun_out/prof_gemm_full python tools/one_step.py > /dev/null 2>&1
python tools/gemm_full_summary.py gpurun_out/prof_gemm_full.ncu-rep gpurun_out/prof_ncu_summary.json > gpurun_out/prof_gemm_full.txt
cat gpurun_out/prof_launches.txt | head -12
cat gpurun_out/prof_gemm_full.txt
