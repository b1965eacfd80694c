timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "^(FAILED|E  )|passed|failed" | head -20
for c in "30 3 C5" "23 5 C2" "23 5 C3" "23 3 C4" "17 5 C1" "23 3 D1"; do timeout 300 python tools/c5_probe.py $c 2>&1 | tail -1; done
