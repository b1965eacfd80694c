# encoder occupancy: __launch_bounds__(256, HUSKY_ENC_MINB)
B='import importlib.util
spec=importlib.util.spec_from_file_location("b","paper_2012_00866_b200/_build.py"); b=importlib.util.module_from_spec(spec); spec.loader.exec_module(b); b.build(force=True)'
HUSKY_NVCC_DEFS="-DHUSKY_ENC_MINB=5" python -c "$B" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py -x -q -k "not multi" > gpurun_out/pytest_e.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_e.log
for rep in 1 2; do for v in 1 4 5 6; do
  HUSKY_NVCC_DEFS="-DHUSKY_ENC_MINB=$v" python -c "$B" > /dev/null 2>&1 || echo build failed
  for c in C2 C3; do TAG=minb$v timeout 120 python tools/lab_sort.py $c | sed 's/stages.*encode.: \([0-9.]*\).*/encode \1/'; done
done; done 2>&1 | tee gpurun_out/lab_enc.txt
python -c "$B" > /dev/null 2>&1
