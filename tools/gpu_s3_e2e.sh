# host_many with depth + 1 output slots: its GPU tests, then the C5 bench line (e2e) without the extras
python -c "import torch; f,t=torch.cuda.mem_get_info(); print('mem free/total GB', f/1e9, t/1e9)"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "host" -p no:cacheprovider 2>&1 | tail -2
timeout 900 python bench.py --no-also --no-cpu-baseline --no-library-bar > gpurun_out/s3_e2e.json 2> gpurun_out/s3_e2e.err; echo bench=$?
tail -3 gpurun_out/s3_e2e.err
python -c "
import json; d=json.loads(open('gpurun_out/s3_e2e.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], json.dumps(d.get('e2e')))"
