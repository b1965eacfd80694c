python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next.py tests/test_gpu_keysort.py tests/test_gpu_infra.py -x -q 2>&1 | tail -4
for c in "30 3 C5" "23 5 C2" "23 5 C3" "17 5 C1" "23 3 C4"; do timeout 300 python tools/c5_probe.py $c 2>&1 | tail -1; done
