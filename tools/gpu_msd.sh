python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_keysort.py -x -q > gpurun_out/pytest_keysort.log 2>&1; echo keysort=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
for c in C2 C3 C1 C4; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_msd_$c.json 2> gpurun_out/bench_msd_$c.err; echo bench $c=$?; done
HUSKY_KEYSORT=lsd timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_lsd_C2.json 2> gpurun_out/bench_lsd_C2.err; echo lsd=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_msd.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo ncu=$?
