# split-K sweep of the batched path at 128 sessions
for q in 1 2 3; do for o in 3 6 9; do
  echo "KSQ=$q KSO=$o $(EKV_BATCH_KSQ=$q EKV_BATCH_KSO=$o timeout 120 python tools/bench_batch.py --sessions 128 2>&1 | tail -1 | cut -c1-60)"
done; done
