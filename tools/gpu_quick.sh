# quick check: build + GPU parity subset + C2/C3/C4 timing of the working tree
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_next.py tests/test_gpu_keysort.py -x -q > gpurun_out/pytest_q.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_q.log
for c in ${CONFIGS:-C2 C3 C4}; do TAG=q timeout 120 python tools/lab_sort.py $c; done 2>&1 | tee gpurun_out/lab_quick.txt
