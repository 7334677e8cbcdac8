timeout 300 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -2
for pf in 0 8 16 32 64 128 256; do
  EKV_MEGA_PREFETCH=$pf timeout 200 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/pf.json 2> gpurun_out/pf.err
  python -c "
import json;d=json.load(open('gpurun_out/pf.json'));print('PF $pf', round(d['value']), round(d['ms_per_step']*1000,1), 'us', round(d['roofline']['frac'],3))"
done
