# Plain bench, then (only after it exits 0) the launch list and one full capture
# of each kernel of the path.  Usage: bash tools/ncu_round.sh <tag>
set -e
T=${1:-cur}
python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/${T}_plain.json 2> gpurun_out/${T}_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_step -s 10 -c 1 -o gpurun_out/${T}_mega python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_ncu_mega.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:kv_compress_tile -c 1 -o gpurun_out/${T}_k3 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_ncu_k3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:align_qnorm -c 1 -o gpurun_out/${T}_k1 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_ncu_k1.log 2>&1
echo done
