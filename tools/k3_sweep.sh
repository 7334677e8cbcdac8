for c in "" ""; do
  EKV_K3_CFG=$c timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-concurrency --no-c4 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); a=d['align_compress']; print('cfg=$c', 'K3', round(a['k3_ms']*1000,1), 'us', round(a['k3_gbs']), round(a['k3_frac'],3))"
done
