# A/B of the working tree against the previous versions of some csrc files on
# one box: tools/ab_prev/<name> replaces paper_2012_00866_b200/csrc/<name> for
# the "prev" builds.  CONFIGS (default "C2 C3") are timed with tools/lab_sort.py.
B='import importlib.util
spec=importlib.util.spec_from_file_location("b","paper_2012_00866_b200/_build.py"); b=importlib.util.module_from_spec(spec); spec.loader.exec_module(b); b.build(force=True)'
C=paper_2012_00866_b200/csrc
mkdir -p /tmp/ab_new
for f in tools/ab_prev/*; do cp $C/$(basename $f) /tmp/ab_new/; done
for v in new prev new prev; do
  for f in tools/ab_prev/*; do
    if [ $v = prev ]; then cp $f $C/$(basename $f); else cp /tmp/ab_new/$(basename $f) $C/; fi
  done
  python -c "$B" > /dev/null 2>&1 || echo build failed
  for c in ${CONFIGS:-C2 C3}; do TAG=$v timeout 120 python tools/lab_sort.py $c; done
done 2>&1 | tee gpurun_out/lab_ab.txt
for f in tools/ab_prev/*; do cp /tmp/ab_new/$(basename $f) $C/; done
python -c "$B" > /dev/null 2>&1
