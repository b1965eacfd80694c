# round-end refresh: full GPU tests + smoke, bench C1-C4 (+ reference arm, + sharded path), ncu evidence
bash tools/gpu_tests.sh
bash tools/gpu_bench_ncu.sh
for x in peer nccl; do HUSKY_EXCHANGE=$x timeout 300 python bench.py --force-multi --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_fm_$x.json 2> gpurun_out/bench_fm_$x.err; echo fm $x=$?; done
