# compute-sanitizer over every step variant; summaries in gpurun_out/sanitize/.
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for v in plain debug adaptive rotate airpf1 airpf2 multinomial sharded-pairwise sharded-pull sharded-peer; do
  for t in memcheck racecheck synccheck initcheck; do
    timeout 600 $CS --tool $t --error-exitcode 9 --print-limit 20 python tools/sanitize_run.py $v \
      > gpurun_out/sanitize/${v}_${t}.log 2>&1
    echo "$v $t rc=$?" >> gpurun_out/sanitize/summary.txt
  done
done
