# Round measurement: plain bench with CPU baseline, the reference arm, then -- each only after
# the plain run exited 0 -- the launch list and one full capture per kernel of the path
# (decode megakernel, K3, K1, the batched K9/K10/K11, the prefill's K10).
# Usage: bash tools/ncu_round2.sh <tag>
set -e
T=${1:-cur}
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python bench.py --impl reference > gpurun_out/${T}_reference.json 2> gpurun_out/${T}_reference.err
Q="--steps 30 --warmup 5 --no-cpu-baseline --no-c4"
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-concurrency --no-c4 > gpurun_out/${T}_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_step -s 10 -c 1 -o gpurun_out/${T}_mega python bench.py $Q --no-concurrency > gpurun_out/${T}_ncu_mega.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:kv_compress_tile_kernelILi128 -c 1 -o gpurun_out/${T}_k3 python bench.py $Q --no-concurrency > gpurun_out/${T}_ncu_k3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:align_qnorm -c 1 -o gpurun_out/${T}_k1 python bench.py $Q --no-concurrency > gpurun_out/${T}_ncu_k1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:batch_ -s 300 -c 5 -o gpurun_out/${T}_batch python tools/bench_batch.py --sessions 128 --steps 2 --warmup 1 > gpurun_out/${T}_ncu_batch.log 2>&1
echo done
