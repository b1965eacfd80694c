python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -k "staged or fix or run or off_domain or general or fuzz" 2>&1 | tail -2
for c in "23 3 D1" "20 3 D1"; do timeout 300 python tools/c5_probe.py $c 2>&1 | tail -1; done
