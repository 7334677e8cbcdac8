T=${1:-b}
timeout 600 python -m pytest tests/test_gpu_batch.py -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${T}_pytest.log
timeout 300 python tools/bench_batch.py --sessions ${2:-1,64,128,256} 2>&1 | tail -8
