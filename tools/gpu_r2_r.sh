python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "slab or C1 or C2 or C3 or C5 or alphabet" 2>&1 | tail -2
for c in "30 3 C5" "23 5 C2" "23 5 C3"; do timeout 300 python tools/c5_probe.py $c 2>&1 | tail -1; done
