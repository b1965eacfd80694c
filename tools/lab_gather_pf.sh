# gather: exact packed lengths + where the long strings' prefetch goes (HUSKY_GATHER_PF 0/1/2) vs tools/ab_prev
B='import importlib.util
spec=importlib.util.spec_from_file_location("b","paper_2012_00866_b200/_build.py"); b=importlib.util.module_from_spec(spec); spec.loader.exec_module(b); b.build(force=True)'
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_next.py -x -q > gpurun_out/pytest_g.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_g.log
for rep in 1 2; do
for v in 0 1 2; do
  HUSKY_NVCC_DEFS="-DHUSKY_GATHER_PF=$v" python -c "$B" > /dev/null 2>&1 || echo build failed
  for c in C2 C3; do TAG="pf$v" timeout 120 python tools/lab_sort.py $c | sed 's/stages.*radix_pass.: \([0-9.]*\).*gather.: \([0-9.]*\).*/radix \1 gather \2/'; done
done
done 2>&1 | tee gpurun_out/lab_gather_pf.txt
CONFIGS="C2 C3" bash tools/lab_ab.sh | sed 's/stages.*gather.: \([0-9.]*\).*/gather \1/'
