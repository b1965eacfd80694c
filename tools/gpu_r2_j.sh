timeout 300 python tools/c5_probe.py 20 2 D1 > gpurun_out/probe_d1.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fix_staged" -s 1 -c 1 -o gpurun_out/r2j_fix python tools/c5_probe.py 20 2 D1 > gpurun_out/ncu_j.log 2>&1; echo ncu=$?
