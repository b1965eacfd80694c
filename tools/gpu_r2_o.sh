python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_large.py -x -q 2>&1 | tail -2
N=268447801
timeout 300 python tools/c5_probe.py $N 1 > gpurun_out/probe_big.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c5big.csv python tools/c5_probe.py $N 1 > gpurun_out/ncu_l.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gather|k_onesweep|k_encode|k_hist_slots" -s 13 -c 4 -o gpurun_out/r2_full_c5big python tools/c5_probe.py $N 1 > gpurun_out/ncu_f.log 2>&1; echo full=$?
