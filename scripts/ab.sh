#!/bin/bash
# A/B variants on one GPU call: each argument is a quoted list of nvcc -D flags
# (or "base"); every variant is built in-tree and timed by ab_time.py, the
# list twice in alternating order.  Outputs under gpurun_out/ab.
mkdir -p gpurun_out/ab
for pass in 1 2; do
  for v in "$@"; do
    flags=""; [ "$v" != "base" ] && flags="$v"
    python - "$flags" <<'PY'
import sys
from paper_1903_10741_b200 import build as b
b.build(force=True, extra=sys.argv[1].split())
PY
    python scripts/ab_time.py "$v" 300 100 | tee -a gpurun_out/ab/results.jsonl
  done
done
python -c "from paper_1903_10741_b200 import build as b; b.build(force=True)"
