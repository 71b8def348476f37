#!/bin/bash
# Tuning sweep of the tile/CTA knobs (prints ms per launch of each kernel).
N=${N:-67108864}
run() {
  echo "== $*"
  env "$@" python bench.py --N $N --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), {k: v['ms_per_launch'] for k, v in d['kernels'].items()})"
}
for cfg in "$@"; do run $cfg; done
