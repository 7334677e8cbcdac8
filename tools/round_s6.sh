# Final validation of the round at the current tree: GPU tests, smoke, bench (N=1), reference arm,
# launch list and the ncu captures.  Usage: bash tools/round_s6.sh <tag>
T=${1:-r01s6}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"
tail -2 gpurun_out/${T}_smoke.log
timeout 1500 bash tools/ncu_round2.sh ${T}; echo "ncu_round rc=$?"
