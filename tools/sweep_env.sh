# A/B sweep over tuning environment knobs on one box: one bench line per variant.
# usage: VARIANTS_FILE=tools/x.txt TAG=e bash tools/sweep_env.sh   (one "NAME ENV=.. ENV=.." per line)
mkdir -p gpurun_out
T=${TAG:-sw}
out=gpurun_out/${T}_sweep.txt
: > $out
while read -r name rest; do
  [ -z "$name" ] && continue
  envs=""; args=""
  for tok in $rest; do case $tok in *=*) envs="$envs $tok";; *) args="$args $tok";; esac; done
  case $name in *_nows) envs="$envs PF_STAGE_WS=0";; esac
  env $envs timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} $args > gpurun_out/${T}_${name}.json 2> gpurun_out/${T}_${name}.err
  python - "$name" "gpurun_out/${T}_${name}.json" >> $out <<'PY'
import json, sys
name, f = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    ks = " ".join(f"{k}={v['ms_per_launch']:.4f}x{v['launches']}" for k, v in d["kernels"].items())
    print(f"{name:28s} {d['ms_per_step']:.4f} ms/step  {ks}")
except Exception as e:
    print(f"{name:28s} FAILED {e}")
PY
done < ${VARIANTS_FILE}
