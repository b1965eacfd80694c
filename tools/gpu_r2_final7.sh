# final evidence of HEAD: build + smoke, GPU suite, default bench line, reference arm, sharded line, launch list
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/k_build.log 2>&1 || { tail -20 gpurun_out/k_build.log; exit 1; }
tail -1 gpurun_out/k_build.log
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/k_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/k_pytest.log
timeout 1200 python bench.py > gpurun_out/k_bench.json 2> gpurun_out/k_bench.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/k_ref.json 2> gpurun_out/k_ref.err; echo ref=$?
timeout 600 python bench.py --force-multi --n 134217728 --steps 5 --warmup 3 --no-cpu-baseline --no-also > gpurun_out/k_fm.json 2> gpurun_out/k_fm.err; echo fm=$?
KR='regex:^k_(encode|hist_slots|onesweep|radix_finalize|gather|runs_classify|fix_staged|fix_small|fix_medium|regather_runs)'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" -c 60 --csv --log-file gpurun_out/k_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-also --no-e2e --no-library-bar > gpurun_out/k_ncu.log 2>&1; echo launches=$?
