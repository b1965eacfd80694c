# The checked build (HUSKY_CHECKED: kernels count out-of-bounds output / random-read
# indices, never trapping) over the sanitizer case list and the GPU suite -- the
# stand-in for compute-sanitizer memcheck, closed on this pool (profiles/r02_sanitizer.txt).
# HUSKY_CHK_SELFTEST=1 shrinks the bounds by one: the same cases must then FAIL.
set -u
LIBC=paper_2012_00866_b200/libhusky_checked.so
HUSKY_NVCC_DEFS=-DHUSKY_CHECKED python -c "
import importlib.util
spec = importlib.util.spec_from_file_location('b', 'paper_2012_00866_b200/_build.py')
b = importlib.util.module_from_spec(spec); spec.loader.exec_module(b)
print(b.build(out='$LIBC'))" > gpurun_out/checked_build.log 2>&1 || { echo build failed; tail gpurun_out/checked_build.log; exit 1; }
python -c "import __graft_entry__ as g; g.build()" >> gpurun_out/checked_build.log 2>&1
HUSKY_LIB=$LIBC timeout 900 python tools/sanitize_cases.py > gpurun_out/checked_cases.log 2>&1; echo cases=$?
tail -3 gpurun_out/checked_cases.log
HUSKY_LIB=$LIBC HUSKY_CHK_SELFTEST=1 timeout 900 python tools/sanitize_cases.py > gpurun_out/checked_selftest.log 2>&1; echo selftest=$? "(expected nonzero)"
grep -m2 "checked build" gpurun_out/checked_selftest.log
HUSKY_LIB=$LIBC timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/checked_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/checked_pytest.log
# the sharded path's phases at 2^27 C5 strings through a one-rank communicator
HUSKY_MULTI_TIMING=1 timeout 300 python tools/multi_probe.py 27 > gpurun_out/multi_probe27.log 2>&1; echo multi_probe=$?
tail -30 gpurun_out/multi_probe27.log
