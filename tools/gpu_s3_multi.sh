# the sharded path (one-rank NCCL communicator): C5 2^27 with the pipelined e2e, and C2 (1e7) vs husky_sort
timeout 900 python bench.py --force-multi --n 134217728 --steps 5 --warmup 3 --no-cpu-baseline --no-also > gpurun_out/s3_fm27.json 2> gpurun_out/s3_fm27.err; echo fm27=$?
tail -3 gpurun_out/s3_fm27.err
python -c "
import json; d=json.loads(open('gpurun_out/s3_fm27.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['validation'], json.dumps(d.get('e2e')))"
timeout 600 python bench.py --force-multi --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-also --no-e2e > gpurun_out/s3_fmC2.json 2> gpurun_out/s3_fmC2.err; echo fmC2=$?
python -c "
import json; d=json.loads(open('gpurun_out/s3_fmC2.json').read().strip().splitlines()[-1]); print('C2 multi', d['value'], d['ms_per_step'], d['validation'])"
timeout 600 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-also --no-e2e --no-library-bar > gpurun_out/s3_C2.json 2> gpurun_out/s3_C2.err; echo C2=$?
python -c "
import json; d=json.loads(open('gpurun_out/s3_C2.json').read().strip().splitlines()[-1]); print('C2 single', d['value'], d['ms_per_step'])"
