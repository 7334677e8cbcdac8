set -e
python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/mega_plain.json 2> gpurun_out/mega_plain.err
ncu --set full --clock-control none --import-source on -k regex:decode_step -s 10 -c 1 -o gpurun_out/mega python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_mega.log 2>&1
echo done
