T=${1:-bn}
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launch.csv python tools/bench_batch.py --sessions ${2:-128} --steps 2 --warmup 1 > gpurun_out/${T}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:batch_ctx_attn -s 3 -c 1 -o gpurun_out/${T}_k10 python tools/bench_batch.py --sessions ${2:-128} --steps 2 --warmup 1 > gpurun_out/${T}_k10.log 2>&1
echo done
