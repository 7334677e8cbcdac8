# A/B of the persistent decode kernel: tok/s of bench.py's decode (500 steps) per setting
for v in "$@"; do
  for i in 1 2; do
    env $v python bench.py --steps 500 --warmup 20 --no-concurrency --no-c4 --no-c5 --no-c1 --no-e2e-full --no-cpu-baseline 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']), round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_us'],1))"
  done
done
