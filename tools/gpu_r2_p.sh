N=268447801
timeout 300 python tools/c5_probe.py $N 1 > gpurun_out/probe_big.log 2>&1 || exit 1
for k in k_gather k_encode k_hist_slots; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 1 -c 1 -o gpurun_out/r2_full_$k python tools/c5_probe.py $N 1 > gpurun_out/ncu_$k.log 2>&1; echo $k=$?
done
