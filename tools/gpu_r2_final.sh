# round-2 evidence refresh: build + smoke, GPU tests, C5 bench (+ also), reference arm,
# sharded line (one-rank NCCL), ncu launch list of the bench, ncu --set full of the
# top kernels on the 2^30 code path at 2^28 + 12345 strings
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f_build.log 2>&1 || { tail -20 gpurun_out/f_build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/f_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/f_pytest.log
timeout 1200 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f_ref.json 2> gpurun_out/f_ref.err; echo ref=$?
timeout 600 python bench.py --force-multi --n 134217728 --steps 5 --warmup 3 --no-cpu-baseline --no-also > gpurun_out/f_fm.json 2> gpurun_out/f_fm.err; echo fm=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-also --no-e2e --no-library-bar > gpurun_out/f_ncu.log 2>&1; echo launches=$?
for k in k_onesweep k_gather k_encode k_hist_slots; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 -o gpurun_out/f_full_$k -f python tools/c5_probe.py 268447801 1 > gpurun_out/f_ncu_$k.log 2>&1; echo full $k=$?
done
