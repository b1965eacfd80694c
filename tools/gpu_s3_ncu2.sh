# ncu --set full of the kernels changed in the last session (histograms + plan, small fix-up) on the 2^30 code path at 2^28 + 12345
for k in k_hist_slots k_fix_small; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/s3_full_$k -f python tools/c5_probe.py 268447801 1 > gpurun_out/s3_ncu_$k.log 2>&1; echo full $k=$?
  python tools/ncu_summary.py gpurun_out/s3_full_$k.ncu-rep 2>&1 | tail -2
done
