# NEXT-2 check: multi-GPU tests (loopback peer/copy, 1-rank NCCL window/send-recv),
# then the 1-GPU sharded bench through both transports.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -k "multi" -x -q > gpurun_out/pytest_peer.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest_peer.log
for x in peer nccl; do
  HUSKY_EXCHANGE=$x timeout 300 python bench.py --force-multi --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_fm_$x.json 2> gpurun_out/bench_fm_$x.err; echo bench $x=$?
  tail -c 600 gpurun_out/bench_fm_$x.json; echo
  HUSKY_EXCHANGE=$x HUSKY_MULTI_TIMING=1 timeout 300 python bench.py --force-multi --steps 2 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | grep "husky multi" | tail -12
done
