timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "lowest_digit or tiny" 2>&1 | grep -E "^(FAILED|E  )|passed|failed" | head -30
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "^(FAILED|E  )|passed|failed" | head -30
