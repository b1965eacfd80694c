# lean-register onesweep at 2 / 3 CTAs per SM vs the previous kernel (tools/ab_prev)
B='import importlib.util
spec=importlib.util.spec_from_file_location("b","paper_2012_00866_b200/_build.py"); b=importlib.util.module_from_spec(spec); spec.loader.exec_module(b); b.build(force=True)'
C=paper_2012_00866_b200/csrc
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_keysort.py tests/test_gpu_fuzz.py -x -q > gpurun_out/pytest_r.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_r.log
HUSKY_NVCC_DEFS="-DHUSKY_RADIX_MINB=3" python -c "$B" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_keysort.py -x -q > gpurun_out/pytest_r3.log 2>&1; echo pytest3=$?; tail -2 gpurun_out/pytest_r3.log
mkdir -p /tmp/ab_new; cp $C/radix.cu $C/kernels.cuh /tmp/ab_new/
for rep in 1 2; do for v in new2 new3 prev; do
  if [ $v = prev ]; then cp tools/ab_prev/radix.cu tools/ab_prev/kernels.cuh $C/; D=""; else cp /tmp/ab_new/radix.cu /tmp/ab_new/kernels.cuh $C/; D="-DHUSKY_RADIX_MINB=${v#new}"; fi
  HUSKY_NVCC_DEFS="$D" python -c "$B" > /dev/null 2>&1 || echo build failed
  for c in C2 C3; do TAG=$v timeout 120 python tools/lab_sort.py $c | sed 's/stages.*radix_pass.: \([0-9.]*\).*gather.: \([0-9.]*\).*/radix \1 gather \2/'; done
done; done 2>&1 | tee gpurun_out/lab_minb.txt
cp /tmp/ab_new/radix.cu /tmp/ab_new/kernels.cuh $C/; python -c "$B" > /dev/null 2>&1
