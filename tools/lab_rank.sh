python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in C2 C3; do
  for m in 0 1 2 4 8 16 32 64 128 255; do HUSKY_RANK_BALLOT=$m TAG=mask$m python tools/lab_sort.py $c; done
done 2>&1 | tee gpurun_out/lab_rank.txt
