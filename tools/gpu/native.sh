timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_step_native.py 2>&1 | tail -3
python tools/e2e_timeline.py
for v in 1 0; do DIPPM_NATIVE_GRAPHED=$v timeout 600 python bench.py --no-infer --no-fp32 --no-cfg0 --no-cpu-baseline --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('graphed=$v', d['ms_per_step'], d['value'], 'e2e', d['e2e']['value'])"; done
