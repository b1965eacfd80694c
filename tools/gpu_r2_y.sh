timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "slab or lowest or tiny or staged" 2>&1 | grep -E "^(FAILED|E  )|passed|failed" | head -20
for c in "30 3 C5" "26 3 C5"; do timeout 300 python tools/c5_probe.py $c 2>&1 | tail -1; HUSKY_PART=0 timeout 300 python tools/c5_probe.py $c 2>&1 | tail -1; done
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "^(FAILED|E  )|passed|failed" | head -20
