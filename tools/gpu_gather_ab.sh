python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_next.py -x -q > gpurun_out/pytest_g.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_g.log
CONFIGS="C2 C3 C4" bash tools/lab_ab.sh
