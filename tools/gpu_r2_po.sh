timeout 900 python bench.py --no-also --no-library-bar --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/po_c5.json 2> gpurun_out/po_c5.err; echo c5=$?
timeout 300 python bench.py --config C2 --no-library-bar --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/po_c2.json 2> gpurun_out/po_c2.err; echo c2=$?
