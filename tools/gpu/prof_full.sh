# Full ncu capture (with source) of one bf16 training step's kernels, for reading back with
# ncu -i gpurun_out/prof_full.ncu-rep --page details|source --csv.  Usage: bash tools/gpu/prof_full.sh [regex]
K=${1:-regex:.}
ncu --profile-from-start off --set full --import-source on --clock-control none -k "$K" \
    -o gpurun_out/prof_full -f python tools/one_step.py > gpurun_out/prof_full.log 2>&1
echo "ncu rc=$?"
