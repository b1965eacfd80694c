KR='regex:^k_(encode|hist_slots|onesweep|radix_finalize|gather|runs_classify|fix_staged|fix_small|fix_medium|regather_runs)'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" -c 60 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-also --no-e2e --no-library-bar > gpurun_out/f_ncu.log 2>&1; echo launches=$?
for k in k_gather k_encode k_hist_slots k_fix_small; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/f_full_$k -f python tools/c5_probe.py 268447801 1 > gpurun_out/f_ncu_$k.log 2>&1; echo full $k=$?
done
