#!/bin/bash
# quick per-kernel timing sweep: env assignments then bench args after "--"
run() {
  local envs=() ; while [ "$1" != "--" ]; do envs+=("$1"); shift; done; shift
  echo "== ${envs[*]} $*"
  env "${envs[@]}" timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), '%.3g'%d['value'], {k: (v['ms_per_launch'], v['launches']) for k, v in d['kernels'].items()})" 2>&1
}
while read -r line; do
  [ -z "$line" ] && continue
  case "$line" in \#*) continue;; esac
  eval run $line
done < ${CASES:-tools/sweep_cases.txt}
