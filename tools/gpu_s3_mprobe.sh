HUSKY_MULTI_TIMING=1 timeout 300 python tools/multi_probe.py 23 > gpurun_out/mprobe23_t.log 2>&1; echo t=$?
grep "husky multi" gpurun_out/mprobe23_t.log | tail -11
timeout 300 python tools/multi_probe.py 23 > gpurun_out/mprobe23.log 2>&1; echo p=$?
cat gpurun_out/mprobe23.log | grep -v NCCL
