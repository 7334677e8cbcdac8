timeout 300 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -2
timeout 100 python tools/trace_mega.py
timeout 200 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/q.json 2> gpurun_out/q.err
python -c "
import json;d=json.load(open('gpurun_out/q.json'));print('BENCH', d['value'],d['ms_per_step'],d['roofline']['frac'],d['e2e']['value'])"
