for i in 1 2 3; do
  timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-concurrency > gpurun_out/c4r.json 2>/dev/null
  python -c "
import json;c=json.load(open('gpurun_out/c4r.json'))['long_context_pipeline'];print('c4', round(c['sequential_ms'],1), round(c['pipelined_ms'],1), round(c['overlap_efficiency'],2))"
done
