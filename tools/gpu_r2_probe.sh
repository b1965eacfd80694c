set -x
nproc; free -g; lscpu | grep -i "model name\|socket\|numa node(s)"; nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests/test_gpu_infra.py -x -q 2>&1 | tail -5
timeout 600 python tools/c5_probe.py 30 3 > gpurun_out/c5_probe_lsd.json 2> gpurun_out/c5_probe_lsd.err; tail -3 gpurun_out/c5_probe_lsd.err
HUSKY_KEYSORT=msd timeout 600 python tools/c5_probe.py 30 3 > gpurun_out/c5_probe_msd.json 2> gpurun_out/c5_probe_msd.err; tail -3 gpurun_out/c5_probe_msd.err
cat gpurun_out/c5_probe_*.json
