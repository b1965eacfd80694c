python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for hnt in 0 1 2 3; do HUSKY_RADIX_HINTS=$hnt TAG=hints$hnt python tools/lab_sort.py C2; done 2>&1 | tee gpurun_out/lab_hints.txt
TAG=hints0-C3 python tools/lab_sort.py C3 | tee -a gpurun_out/lab_hints.txt
HUSKY_RADIX_HINTS=3 TAG=hints3-C3 python tools/lab_sort.py C3 | tee -a gpurun_out/lab_hints.txt
