python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -4 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-C2 C3 C4}; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench $c=$?; python - <<PY
import json; d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$c', d['value'], d['ms_per_step'], 'radix', r['frac'], 'enc', r['encode']['frac'], {k:v['ms_per_step'] for k,v in d['stages'].items()})
PY
done
