#!/bin/bash
# ncu --set full captures (with source) of the three GA-step kernels in the bench's launch configuration.
TAG=${1:-p}
mkdir -p gpurun_out/$TAG
for k in order_warp_kernel lane_decode2_kernel generation_kernel; do
  ncu --set full --import-source on --clock-control none -k regex:"$k" -s 4 -c 1 -o gpurun_out/$TAG/$k python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
ls gpurun_out/$TAG
