# programmatic dependent launch of the radix pass slots: HUSKY_PDL=1 (default) vs 0
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_keysort.py tests/test_gpu_fuzz.py -x -q > gpurun_out/pytest_pdl.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_pdl.log
for rep in 1 2; do for v in 1 0; do
  for c in C2 C3; do HUSKY_PDL=$v TAG="pdl$v" timeout 120 python tools/lab_sort.py $c | sed 's/stages.*radix_pass.: \([0-9.]*\).*gather.: \([0-9.]*\).*/radix \1 gather \2/'; done
done; done 2>&1 | tee gpurun_out/lab_pdl.txt
