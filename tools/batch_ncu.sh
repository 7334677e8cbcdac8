ncu --metrics gpu__time_duration.sum --clock-control none -k regex:batch -c 400 --csv --log-file gpurun_out/bl128.csv python tools/bench_batch.py --sessions 128 --steps 2 --warmup 1 > gpurun_out/bl128.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:batch -c 400 --csv --log-file gpurun_out/bl1024.csv python tools/bench_batch.py --sessions 1024 --steps 2 --warmup 1 > gpurun_out/bl1024.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:batch_ctx_attn -s 40 -c 2 -o gpurun_out/k10_128 python tools/bench_batch.py --sessions 128 --steps 2 --warmup 1 > gpurun_out/k10n.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:batch_user_merge -s 40 -c 1 -o gpurun_out/k11_128 python tools/bench_batch.py --sessions 128 --steps 2 --warmup 1 > gpurun_out/k11n.log 2>&1
echo ok
