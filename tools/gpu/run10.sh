for i in 1 2 3; do timeout 900 python -m pytest tests -m gpu -q 2>&1 | grep -E "passed|failed|^FAILED|^E  " | head -8; done
timeout 600 python bench.py --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r1s2_bench10.json
python -c "
import json; d=json.load(open('gpurun_out/r1s2_bench10.json'))
print('value', d['value'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'], 'ms', d['ms_per_step'])
print(json.dumps(d['inference']['predict_from_json'], indent=1))"
