# usage: bash tools/sweep_env.sh VAR v1 v2 ...
VAR=$1; shift
timeout 300 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -1
for v in "$@"; do
  env $VAR=$v timeout 200 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/sw.json 2> gpurun_out/sw.err
  python -c "
import json;d=json.load(open('gpurun_out/sw.json'));print('$VAR=$v', round(d['value']), round(d['ms_per_step']*1000,1), 'us', round(d['roofline']['frac'],3))"
done
