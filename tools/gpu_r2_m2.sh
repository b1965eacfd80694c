timeout 600 python bench.py --n 134217728 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-also --no-library-bar > gpurun_out/b27_single.json 2> gpurun_out/b27_single.err; echo single=$?
timeout 600 python bench.py --force-multi --n 134217728 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-also > gpurun_out/b27_multi.json 2> gpurun_out/b27_multi.err; echo multi=$?
