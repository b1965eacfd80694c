# husky_sort_host_many: three-stream pipeline (default) vs worker threads (HUSKY_HOST_MANY=threads)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for m in pipe threads; do HUSKY_HOST_MANY=$m timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "host" > gpurun_out/pytest_hm_$m.log 2>&1; echo pytest $m=$?; tail -1 gpurun_out/pytest_hm_$m.log; done
for rep in 1 2; do for m in pipe threads; do for d in 2 3; do
  HUSKY_HOST_MANY=$m HUSKY_E2E_DEPTH=$d timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$m depth $d', d['e2e']['value'], d['e2e']['ms_per_step'])"
done; done; done 2>&1 | tee gpurun_out/lab_hostmany.txt
