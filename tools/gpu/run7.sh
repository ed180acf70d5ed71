timeout 600 python -m pytest tests/test_gpu_scale.py -x -q 2>&1 | tail -3
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/r1s2_bench7.json
python -c "
import json; d=json.load(open('gpurun_out/r1s2_bench7.json'))
print('value', d['value'], 'e2e', d['e2e'], 'frac', d['roofline']['frac'], 'ms', d['ms_per_step'])
print('infer', d['inference'])"
