python -c "import __graft_entry__ as g; g.build()"
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_next.py tests/test_gpu_keysort.py -x -q 2>&1 | tail -3
for c in "17 5 C1" "10 5 C1" "13 5 C1" "16 5 C2"; do timeout 300 python tools/c5_probe.py $c 2>&1 | tail -1; done
for c in "17 5 C1" "10 5 C1"; do HUSKY_SMALL=0 timeout 300 python tools/c5_probe.py $c 2>&1 | tail -1; done
