# onesweep fine-tuning: keys per thread (HUSKY_RADIX_ITEMS) x look-back window (RADIX_LB_W)
B='import importlib.util
spec=importlib.util.spec_from_file_location("b","paper_2012_00866_b200/_build.py"); b=importlib.util.module_from_spec(spec); spec.loader.exec_module(b); b.build(force=True)'
for rep in 1; do for it in 12 14; do for lw in 10 12 14 16; do
  HUSKY_NVCC_DEFS="-DHUSKY_RADIX_ITEMS=$it -DRADIX_LB_W=$lw" python -c "$B" > /dev/null 2>&1 || echo build failed
  for c in C2 C3; do TAG="it$it-w$lw" timeout 120 python tools/lab_sort.py $c | sed 's/stages.*radix_pass.: \([0-9.]*\).*/radix \1/'; done
done; done; done 2>&1 | tee gpurun_out/lab_tune.txt
python -c "$B" > /dev/null 2>&1
