timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_gpu_fuzz.py -x -q -k "slab or C5 or large or fuzz" 2>&1 | grep -E "^(FAILED|E  )|passed|failed" | head -20
for c in "30 3 C5" "26 3 C5" "23 3 C2"; do timeout 300 python tools/c5_probe.py $c 2>&1 | tail -1; done
