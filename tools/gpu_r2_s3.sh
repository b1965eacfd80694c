# session-3 check of HEAD on a fresh box: build + smoke, the GPU suite, the default bench line
bash tools/gpu_tests.sh
timeout 900 python bench.py > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err; echo bench=$?; tail -c 600 gpurun_out/s3_bench.json
