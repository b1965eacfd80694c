HUSKY_EXCHANGE=nccl timeout 300 python tools/multi_probe.py 23 > gpurun_out/mprobe23_nccl.log 2>&1; echo p=$?
cat gpurun_out/mprobe23_nccl.log | grep -v NCCL | grep -v "^radix_pass\|^fix\|^runs"
timeout 300 python tools/c5_probe.py 23 5 C5 2>&1 | tail -1 | cut -c1-700
