timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-library-bar > gpurun_out/l_bench.json 2> gpurun_out/l_bench.err; echo bench=$?
tail -3 gpurun_out/l_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/l_bench.json').read().strip().splitlines()[-1]); print(d['value'])
for k,v in d['also'].items(): print(k, v.get('value'), v.get('ms_per_step'), v.get('validation'))"
