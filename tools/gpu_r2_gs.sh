timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "^(FAILED|E  )|passed|failed" | head -20
timeout 600 python bench.py --config D1 --no-library-bar --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/gs_d1.json 2> gpurun_out/gs_d1.err; echo d1=$?
timeout 600 python bench.py --config C4 --no-library-bar --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/gs_c4.json 2> gpurun_out/gs_c4.err; echo c4=$?
