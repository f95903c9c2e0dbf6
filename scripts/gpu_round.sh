#!/bin/bash
# One GPU session: tests, bench, ncu launch list + full capture of the two
# evaluate kernels.  Outputs under gpurun_out/$TAG.
TAG=${1:-r01}
mkdir -p gpurun_out/$TAG
python -m pytest tests -m gpu -q > gpurun_out/$TAG/pytest_gpu.txt 2>&1; tail -3 gpurun_out/$TAG/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$TAG/smoke.txt 2>&1; tail -1 gpurun_out/$TAG/smoke.txt
python bench.py > gpurun_out/$TAG/bench.json 2> gpurun_out/$TAG/bench.err; tail -2 gpurun_out/$TAG/bench.err; cut -c1-300 gpurun_out/$TAG/bench.json
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/$TAG/bench_ref.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/$TAG/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"lane_decode|order_warp" -s 2 -c 2 -o gpurun_out/$TAG/prof_eval python scripts/prof_eval.py 65536 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"generation_kernel" -s 1 -c 1 -o gpurun_out/$TAG/prof_gen python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out/$TAG
