set -e
python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:kv_compress_tile -c 1 -o gpurun_out/k3 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_k3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 40 -c 2 -o gpurun_out/gemv python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_gemv.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 40 -c 2 -o gpurun_out/attn python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_attn.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:align_qnorm -c 1 -o gpurun_out/k1 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_k1.log 2>&1
echo done
