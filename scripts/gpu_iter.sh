#!/bin/bash
# Perf iteration on one GPU call: GA/evaluate parity tests, the default bench
# line (no cpu baseline), the ncu launch list of a short bench, and ncu --set
# full captures of the named kernels.  usage: gpu_iter.sh TAG "kernel regexes"
TAG=${1:-it}
KERNELS=${2:-generation_kernel}
mkdir -p gpurun_out/$TAG
python -m pytest tests/test_gpu_ga.py tests/test_gpu_fullsize.py::test_config_c_ga_at_bench_launch tests/test_gpu_realwt.py tests/test_gpu_evaluate.py -m gpu -q -x > gpurun_out/$TAG/pytest.txt 2>&1; tail -2 gpurun_out/$TAG/pytest.txt
python bench.py --no-cpu-baseline > gpurun_out/$TAG/bench.json 2> gpurun_out/$TAG/bench.err; tail -2 gpurun_out/$TAG/bench.err
python - gpurun_out/$TAG/bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print({k:d.get(k) for k in ('value','ms_per_step')}, 'eval_only', d.get('eval_only',{}).get('ms_per_launch'), d.get('clocks'))
PY
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/$TAG/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/$TAG/launches.csv 2>/dev/null | head -20
for k in $KERNELS; do
  ncu --set full --import-source on --clock-control none -k regex:"$k" -s 4 -c 1 -o gpurun_out/$TAG/$k python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
ls gpurun_out/$TAG
