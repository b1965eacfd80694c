python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_r2e.json 2> gpurun_out/bench_r2e.err; echo bench rc=$?
timeout 300 python tools/c5_probe.py 28 1 > gpurun_out/probe28e.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_gather" -s 2 -c 1 -o gpurun_out/r2e_gather python tools/c5_probe.py 28 1 > gpurun_out/ncu_e1.log 2>&1; echo ncu1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_encode|k_hist" -s 4 -c 2 -o gpurun_out/r2e_enc python tools/c5_probe.py 28 1 > gpurun_out/ncu_e2.log 2>&1; echo ncu2=$?
