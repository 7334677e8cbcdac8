for i in 1 2; do timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); a=d['align_compress']; print('K3', round(a['k3_ms']*1000,1), 'us', round(a['k3_gbs']), round(a['k3_frac'],3), 'decode', round(d['value']))"; done
