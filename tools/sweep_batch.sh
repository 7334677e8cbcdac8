# split-K sweep of the batched path
for B in 64 128 256; do for q in 1 2 3; do
  echo "B=$B KSQ=$q $(EKV_BATCH_KSQ=$q timeout 120 python tools/bench_batch.py --sessions $B 2>&1 | tail -1 | cut -c1-90)"
done; done
