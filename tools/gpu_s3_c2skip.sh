# C2 / C1 / C5-2^23 with the partial key sort forced (HUSKY_SKIP=2: one digit, 3: two) vs the entropy rule (1)
for sk in 1 2 3 1 2 3; do
  echo "== HUSKY_SKIP=$sk"
  for c in C2 C1; do HUSKY_SKIP=$sk timeout 300 python tools/c5_probe.py 10000000 5 $c 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', [round(x,3) for x in d['ms']], d['stages'].get('radix_pass'), d['stages'].get('fix_small'), d['stages'].get('fix_medium'), d['outcome']['radix_passes'], d['outcome']['n_runs'], d['outcome']['refine_rounds'], d['verify'])"; done
done 2>&1 | tee gpurun_out/s3_c2skip.txt
