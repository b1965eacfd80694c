python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/c5_probe.py 20 2 D1 > gpurun_out/probe_d1.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fix_staged" -s 1 -c 1 -o gpurun_out/r2h_fix python tools/c5_probe.py 20 2 D1 > gpurun_out/ncu_h.log 2>&1; echo ncu=$?
