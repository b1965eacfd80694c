# A/B of two radix.cu versions on one box: the working tree vs tools/radix_prev.cu.txt
B='import importlib.util
spec=importlib.util.spec_from_file_location("b","paper_2012_00866_b200/_build.py"); b=importlib.util.module_from_spec(spec); spec.loader.exec_module(b); b.build(force=True)'
C=paper_2012_00866_b200/csrc
cp $C/radix.cu /tmp/radix_new.cu; cp $C/kernels.cuh /tmp/kernels_new.cuh
for v in new prev new prev; do
  if [ $v = prev ]; then cp tools/radix_prev.cu.txt $C/radix.cu; cp tools/kernels_prev.cuh.txt $C/kernels.cuh; else cp /tmp/radix_new.cu $C/radix.cu; cp /tmp/kernels_new.cuh $C/kernels.cuh; fi
  python -c "$B" > /dev/null 2>&1 || echo build failed
  for c in C2 C3; do TAG=$v timeout 120 python tools/lab_sort.py $c; done
done 2>&1 | tee gpurun_out/lab_ab_radix.txt
cp /tmp/radix_new.cu $C/radix.cu; cp /tmp/kernels_new.cuh $C/kernels.cuh
