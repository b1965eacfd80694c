python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "lowest_digit" 2>&1 | tail -3
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in "30 3 C5" "23 5 C2" "23 5 C3" "17 5 C1"; do timeout 300 python tools/c5_probe.py $c 2>&1 | tail -1; done
