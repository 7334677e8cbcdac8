for i in 1 2; do
  timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline --no-concurrency --no-c4 --no-c5 > gpurun_out/g.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/g.json'));print('run', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['frac'],3))"
done
timeout 600 python -m pytest tests/test_gpu_decode.py -q -x 2>&1 | tail -1
