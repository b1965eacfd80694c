B='import importlib.util
spec=importlib.util.spec_from_file_location("b","paper_2012_00866_b200/_build.py"); b=importlib.util.module_from_spec(spec); spec.loader.exec_module(b); b.build(force=True)'
HUSKY_NVCC_DEFS="-DHUSKY_TIMING" python -c "$B" > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; exit 1; }
for c in C2 C3; do echo "== $c"; HUSKY_PDL=0 python tools/tile_timing.py $c; done 2>&1 | tee gpurun_out/ttiming.txt
python -c "$B" > /dev/null 2>&1
