set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "slab or host_many or C2 or C5" 2>&1 | tail -3
timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-library-bar > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; echo rc=$?
timeout 300 python tools/c5_probe.py 28 1 > gpurun_out/probe28.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gather|k_onesweep|k_encode" -s 3 -c 3 -o gpurun_out/r2_c5_28 python tools/c5_probe.py 28 1 > gpurun_out/ncu_r2.log 2>&1; echo ncu=$?
