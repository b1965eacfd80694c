python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in "30 3 C5" "23 5 C2" "23 5 C3" "17 5 C1" "23 3 C4"; do timeout 300 python tools/c5_probe.py $c 2>&1 | tail -1; done
HUSKY_GRAPH=0 timeout 300 python tools/c5_probe.py 17 5 C1 2>&1 | tail -1
timeout 600 python bench.py --config C1 --no-cpu-baseline --no-e2e --no-library-bar --no-also > gpurun_out/bench_c1.json 2>gpurun_out/bench_c1.err; echo c1 rc=$?
timeout 900 python bench.py --force-multi --no-also > gpurun_out/bench_fm.json 2>gpurun_out/bench_fm.err; echo fm rc=$?
