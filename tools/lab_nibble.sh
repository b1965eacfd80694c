# ranking primitive: ballots / match_any (default rule) vs two 4-bit matches (HUSKY_RANK_NIBBLE 1: spread digits, 2: all, 3: non-spread digits; 4: 3+3+2 bits, 5: 4 x 2 bits, 6: 5+3 bits, 7: ballots everywhere, 9: 3+3 match + 2 ballots, 10: 4+2 match + 2 ballots)
B='import importlib.util
spec=importlib.util.spec_from_file_location("b","paper_2012_00866_b200/_build.py"); b=importlib.util.module_from_spec(spec); spec.loader.exec_module(b); b.build(force=True)'
HUSKY_NVCC_DEFS="-DHUSKY_RANK_NIBBLE=9" python -c "$B" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_keysort.py -x -q -k "not multi" > gpurun_out/pytest_nib.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_nib.log
for rep in 1 2; do for v in 4 9 10; do
  HUSKY_NVCC_DEFS="-DHUSKY_RANK_NIBBLE=$v" python -c "$B" > /dev/null 2>&1 || echo build failed
  for c in C2 C3 C4; do TAG="nib$v" timeout 120 python tools/lab_sort.py $c | sed 's/stages.*radix_pass.: \([0-9.]*\).*/radix \1/'; done
done; done 2>&1 | tee gpurun_out/lab_nibble.txt
python -c "$B" > /dev/null 2>&1
