nproc
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r1s2_bench9.json
python -c "
import json; d=json.load(open('gpurun_out/r1s2_bench9.json'))
print('value', d['value'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'], 'ms', d['ms_per_step'])
print(json.dumps(d['inference'], indent=1))"
