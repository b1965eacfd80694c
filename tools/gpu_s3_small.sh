# small-input look-back: the GPU suite, then A/B (lab/base = HEAD) at C1 1e5, 3e5 and C2 2^23
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/s3_small_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/s3_small_pytest.log
for v in base new base new; do
  if [ $v = base ]; then export HUSKY_LIB=$PWD/lab/base/libhusky.so; else unset HUSKY_LIB; fi
  echo "== $v"
  for n in 1000 100000 300000; do timeout 300 python tools/c5_probe.py $n 7 C1 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['n'], [round(x,4) for x in d['ms']], d['stages'].get('radix_pass'), d['verify'])"; done
  timeout 300 python tools/c5_probe.py 23 5 C2 2>&1 | tail -1 | cut -c1-300
done 2>&1 | tee gpurun_out/s3_small_ab.txt
