#!/bin/bash
# Quick GPU check: parity tests + default bench line.  Outputs under gpurun_out/$TAG.
TAG=${1:-quick}
mkdir -p gpurun_out/$TAG
python -m pytest tests -m gpu -x -q > gpurun_out/$TAG/pytest_gpu.txt 2>&1; tail -3 gpurun_out/$TAG/pytest_gpu.txt
python bench.py ${BENCH_ARGS:---no-cpu-baseline} > gpurun_out/$TAG/bench.json 2> gpurun_out/$TAG/bench.err; tail -2 gpurun_out/$TAG/bench.err
python - <<'PY' gpurun_out/$TAG/bench.json
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print({k:d.get(k) for k in ('value','ms_per_step','gens_per_s')}, 'eval_only', d.get('eval_only'))
PY
if [ -n "$LAUNCHES" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/$TAG/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/$TAG/launches.csv
fi
