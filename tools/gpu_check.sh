# Quick GPU check: full gpu test suite, then a short bench.  Usage: bash tools/gpu_check.sh <tag>
T=${1:-chk}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${T}_pytest.log
timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/${T}_bench.json'));print('BENCH', d['value'],d['ms_per_step'],d['roofline']['frac'],d['e2e']['value'])"
