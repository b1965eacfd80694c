# compute-sanitizer over tools/sanitize_cases.py, ONE tool per gpurun call
# (B200_PROFILING.md): bash tools/gpu_sanitize.sh memcheck|racecheck|synccheck
tool=${1:-memcheck}
python tools/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/sanitize_plain.log; exit 1; }
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
  python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
echo "$tool rc=$?"
tail -5 gpurun_out/sanitize_$tool.log
