for g in 96 128 64 120 128; do
  EKV_MEGA_GRID=$g timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline --no-concurrency --no-c4 > gpurun_out/g.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/g.json'));print('grid=$g', round(d['value'],1), round(d['e2e']['value'],1))"
done
