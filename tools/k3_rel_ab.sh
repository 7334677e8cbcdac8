# RECORD ONLY: the EKV_K3_CFG switch and the per-warp release variants were reverted after
# this A/B (profiles/r01s6_k3_release_ab.txt); the script no longer selects anything.
# A/B of K3 stage release: 0 = CTA barrier (default), 1/2/3 = per-warp mbarrier release with
# 2x8 KB / 3x8 KB / 4x4 KB stages.  Then the K3 parity tests under each setting.
for r in 1 2; do for c in 0 1 2 3; do
  EKV_K3_CFG=$c timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-concurrency --no-c4 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); a=d['align_compress']; s=d['compression_sweep']; print('cfg=$c', 'K3', round(a['k3_ms']*1000,1), 'us', round(a['k3_gbs']), round(a['k3_frac'],3), 'C5', [round(x['compress_frac'],3) for x in s])"
done; done
for c in 1 2 3; do EKV_K3_CFG=$c timeout 600 python -m pytest tests -m gpu -q -x -k "compress or kv or parity" 2>&1 | tail -1; done
