python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in "30 3 C5" "23 3 D1"; do timeout 300 python tools/c5_probe.py $c 2>&1 | tail -1; done
