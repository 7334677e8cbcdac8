for p in "" 8 16 32 ""; do
  EKV_MEGA_PREFETCH=$p timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline --no-concurrency --no-c4 > gpurun_out/g.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/g.json'));print('prefetch=$p', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['frac'],3))"
done
