# small-input tile threshold (HUSKY_RADIX_SMALL_N): sorts of 1e5 .. 3e6 strings with small / large tiles
B='import importlib.util
spec=importlib.util.spec_from_file_location("b","paper_2012_00866_b200/_build.py"); b=importlib.util.module_from_spec(spec); spec.loader.exec_module(b); b.build(force=True)'
python -c "$B" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_keysort.py tests/test_gpu_next.py tests/test_gpu_fuzz.py -x -q > gpurun_out/pytest_sn.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_sn.log
cat > /tmp/sizes.py <<'PY'
import os, sys, numpy as np, torch
sys.path.insert(0, "."); import paper_2012_00866_b200 as h, workloads as W
for n in (100_000, 300_000, 1_000_000, 2_000_000, 4_000_000):
    w = W.make("C2", n); du = torch.from_numpy(w.units).cuda(); do = torch.from_numpy(w.offsets).cuda()
    ws = torch.empty(h.husky_sort_workspace(0, n, w.units.size), dtype=torch.uint8, device="cuda")
    perm = torch.empty(n, dtype=torch.int32, device="cuda"); su = torch.empty(w.units.size + 8, dtype=du.dtype, device="cuda"); so = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    ts = []
    for i in range(15):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record(); h.husky_sort(0, du, do, perm, su, so, ws); b.record(); torch.cuda.synchronize()
        if i >= 5: ts.append(a.elapsed_time(b))
    print(os.environ.get("TAG"), n, round(float(np.median(ts)) * 1e3, 1), "us", flush=True)
PY
for v in 1000000000 0; do HUSKY_NVCC_DEFS="-DHUSKY_RADIX_SMALL_N=$v" python -c "$B" > /dev/null 2>&1; TAG="small_n<$v" python /tmp/sizes.py; done 2>&1 | tee gpurun_out/lab_small_n.txt
python -c "$B" > /dev/null 2>&1
