# gather: where the long strings' units are prefetched (HUSKY_GATHER_PF 0 = L1 before the scan, 1 = L1 after the publish, 2 = none, 3 = L2 after the publish)
B='import importlib.util
spec=importlib.util.spec_from_file_location("b","paper_2012_00866_b200/_build.py"); b=importlib.util.module_from_spec(spec); spec.loader.exec_module(b); b.build(force=True)'
HUSKY_NVCC_DEFS="-DHUSKY_GATHER_PF=3" python -c "$B" > /dev/null 2>&1 || echo build failed
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -k "not multi" > gpurun_out/pytest_g.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_g.log
for rep in 1 2; do for v in 1 3 2; do
  HUSKY_NVCC_DEFS="-DHUSKY_GATHER_PF=$v" python -c "$B" > /dev/null 2>&1 || echo build failed
  for c in C2 C3 C4; do TAG="pf$v" timeout 120 python tools/lab_sort.py $c | sed 's/stages.*gather.: \([0-9.]*\).*/gather \1/'; done
done; done 2>&1 | tee gpurun_out/lab_gather_pf.txt
python -c "$B" > /dev/null 2>&1
