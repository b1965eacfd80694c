timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "refinement_partial or giant or C4 or off_domain" -p no:cacheprovider 2>&1 | tail -3
