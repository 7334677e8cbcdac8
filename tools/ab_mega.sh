timeout 600 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -2
for i in 1 2; do
for v in "" "EKV_MEGA_WO_COLS=1"; do
  env $v timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline --no-concurrency --no-c4 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/ab.json'));print('$v rows' if '$v'=='' else '$v', round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],1))"
done; done
