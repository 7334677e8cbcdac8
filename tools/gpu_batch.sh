T=${1:-b}
timeout 600 python -m pytest tests/test_gpu_batch.py -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/${T}_pytest.log
