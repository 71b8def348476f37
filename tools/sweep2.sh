#!/bin/bash
# quick per-kernel timing sweep: env assignments then bench args after "--"
run() {
  local envs=() ; while [ "$1" != "--" ]; do envs+=("$1"); shift; done; shift
  echo "== ${envs[*]} $*"
  env "${envs[@]}" timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), '%.3g'%d['value'], {k: (v['ms_per_launch'], v['launches']) for k, v in d['kernels'].items()})" 2>&1
}
run X=1 -- --config C4
run PF_INDEX_MODE=0 -- --config C4
run PF_INDEX_MODE=0 PF_MOVE_SMEM=200000 -- --config C4
run PF_INDEX_MODE=0 PF_MOVE_SMEM=60000 -- --config C4
run PF_INDEX_MODE=0 PF_PASS1_SMEM=100000 -- --config C4
run PF_INDEX_MODE=0 PF_PASS1_SMEM=200000 PF_PASS1_THREADS=512 -- --config C4
run X=1 -- --config C2
run PF_INDEX_MODE=0 -- --config C2
run X=1 -- --config C3
run X=1 -- --config C5
run X=1 -- --config C5 --M 2
run X=1 -- --config C5 --M 8192
run X=1 -- --config C1
