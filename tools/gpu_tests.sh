# run a subset of GPU tests: bash tools/gpu_tests.sh <tag> <pytest args...>
T=$1; shift
timeout 900 python -m pytest "$@" -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/${T}_pytest.log
