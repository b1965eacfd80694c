# final check of HEAD: build + smoke, GPU suite, the default bench line, the reference arm
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/h_build.log 2>&1 || { tail -20 gpurun_out/h_build.log; exit 1; }
tail -1 gpurun_out/h_build.log
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/h_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/h_pytest.log
timeout 1200 python bench.py > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/h_ref.json 2> gpurun_out/h_ref.err; echo ref=$?
