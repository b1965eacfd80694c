timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -k "staged or fix or run or lowest or tiny or refinement or fuzz" 2>&1 | grep -E "^(FAILED|E  )|passed|failed" | head -20
for s in 1 2 3; do HUSKY_SKIP=$s timeout 300 python tools/c5_probe.py 23 3 D1 2>&1 | tail -1; done
timeout 300 python tools/c5_probe.py 30 2 C5 2>&1 | tail -1
