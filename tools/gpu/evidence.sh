# Round evidence: bench line, reference arm, launch list, full-step ncu summary, e2e timeline.
timeout 900 python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err; tail -2 gpurun_out/ev_bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 2 > gpurun_out/ev_ref.json 2> gpurun_out/ev_ref.err; tail -1 gpurun_out/ev_ref.json
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ev_launches.csv python tools/one_step.py > /dev/null 2>&1
python tools/ncu_metrics.py gpurun_out/ev_launches.csv > gpurun_out/ev_launches.txt
ncu --profile-from-start off --set full --import-source on --clock-control none -o gpurun_out/ev_step_full -f python tools/one_step.py > /dev/null 2>&1
python tools/ncu_step_summary.py gpurun_out/ev_step_full.ncu-rep gpurun_out/ev_ncu_summary.json > gpurun_out/ev_step_full.txt
python tools/e2e_timeline.py > gpurun_out/ev_e2e_timeline.txt 2>&1
./tools/micro/write_bw > gpurun_out/ev_write_bw.txt 2>&1
cat gpurun_out/ev_launches.txt gpurun_out/ev_step_full.txt gpurun_out/ev_e2e_timeline.txt
