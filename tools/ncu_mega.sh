set -e
python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/v3b_plain.json 2> gpurun_out/v3b_plain.err
ncu --set full --clock-control none --import-source on -k regex:decode_step -s 10 -c 1 -o gpurun_out/v3_mega python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/v3_ncu.log 2>&1
echo done
