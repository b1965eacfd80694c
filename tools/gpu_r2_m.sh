python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 1200 python bench.py > gpurun_out/bench_r2m.json 2> gpurun_out/bench_r2m.err; echo bench rc=$?
timeout 900 python bench.py --force-multi --n 67108864 --no-also > gpurun_out/bench_fm.json 2>gpurun_out/bench_fm.err; echo fm rc=$?
timeout 900 python bench.py --force-multi --config C2 --no-also > gpurun_out/bench_fm_c2.json 2>gpurun_out/bench_fm_c2.err; echo fmc2 rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; echo ref rc=$?
