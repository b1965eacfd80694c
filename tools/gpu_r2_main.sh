set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 900 python bench.py > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; echo rc=$?; tail -5 gpurun_out/bench_r2a.err
