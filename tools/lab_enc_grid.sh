# encoder: strings in flight per thread (HUSKY_ENC_IT) x grid CTAs per SM (HUSKY_ENC_BPS), 4 resident per SM
B='import importlib.util
spec=importlib.util.spec_from_file_location("b","paper_2012_00866_b200/_build.py"); b=importlib.util.module_from_spec(spec); spec.loader.exec_module(b); b.build(force=True)'
for rep in 1 2; do for it in 2 4 8; do for bps in 4 8 16; do
  HUSKY_NVCC_DEFS="-DHUSKY_ENC_IT=$it -DHUSKY_ENC_BPS=$bps" python -c "$B" > /dev/null 2>&1 || echo build failed
  for c in C2 C3; do TAG="it$it-bps$bps" timeout 120 python tools/lab_sort.py $c | sed 's/stages.*encode.: \([0-9.]*\).*/encode \1/'; done
done; done; done 2>&1 | tee gpurun_out/lab_enc_grid.txt
python -c "$B" > /dev/null 2>&1
