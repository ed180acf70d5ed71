# A/B of an env switch on the same box: bench.py (training line only) with and without it.
# usage: bash tools/gpu/ab_bench.sh VAR=value [VAR2=value ...]
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_kernels.py -k "readout" 2>&1 | tail -2
for i in 1 2; do
  timeout 300 python bench.py --no-e2e --no-infer --no-fp32 --no-cfg0 --no-cpu-baseline --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('base', d['ms_per_step'], round(d['roofline']['by_class']['sage_layers_2_3']['us_per_step'],1))"
  env "$@" timeout 300 python bench.py --no-e2e --no-infer --no-fp32 --no-cfg0 --no-cpu-baseline --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*', d['ms_per_step'], round(d['roofline']['by_class']['sage_layers_2_3']['us_per_step'],1))"
done
