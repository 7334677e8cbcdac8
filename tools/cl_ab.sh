for c in "" 4 2 ""; do
  EKV_MEGA_CLUSTER=$c timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline --no-concurrency --no-c4 --no-c5 > gpurun_out/g.json 2> gpurun_out/g.err
  python -c "
import json;d=json.load(open('gpurun_out/g.json'));print('cluster=$c', round(d['value'],1), round(d['e2e']['value'],1))" 2>&1 | tail -1
done
