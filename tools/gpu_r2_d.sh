python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "alphabet or slab or C1 or C5" 2>&1 | tail -2
bash tools/lab_r2_variants.sh
