python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "staged or fix or run or C4 or off_domain or general" 2>&1 | tail -3
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in "23 3 D1" "23 3 C2" "23 3 C4"; do timeout 300 python tools/c5_probe.py $c 2>&1 | tail -1; done
