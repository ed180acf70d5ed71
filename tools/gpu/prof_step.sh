ncu --profile-from-start off --set full --import-source on --clock-control none -o gpurun_out/r2_step_full -f python tools/one_step.py > gpurun_out/r2_step_full.log 2>&1
echo "ncu rc=$?"
python tools/ncu_step_summary.py gpurun_out/r2_step_full.ncu-rep gpurun_out/r2_ncu_summary.json > gpurun_out/r2_step_full.txt 2>&1
cat gpurun_out/r2_step_full.txt
