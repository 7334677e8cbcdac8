for B in 128 256 512; do for q in 0 1; do
  echo "B=$B QFIN=$q $(EKV_BATCH_QFIN=$q timeout 120 python tools/bench_batch.py --sessions $B 2>&1 | tail -1 | cut -c1-80)"
done; done
