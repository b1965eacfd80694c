python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -k "alphabet or slab or C1 or C2 or C5 or fuzz or graph" 2>&1 | tail -2
for c in "30 3 C5" "23 3 C2" "17 5 C1"; do timeout 300 python tools/c5_probe.py $c 2>&1 | tail -1; done
