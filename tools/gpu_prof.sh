#!/bin/bash
# ncu full capture of one kernel: gpu_prof.sh <kernel-regex> <skip> <out-name> <env...> -- <cmd...>
K=$1; SKIP=$2; OUT=$3; shift 3
envs=(); while [ "$1" != "--" ]; do envs+=("$1"); shift; done; shift
mkdir -p gpurun_out
env "${envs[@]}" timeout 600 "$@" > gpurun_out/${OUT}_plain.log 2>&1 && \
env "${envs[@]}" timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 -o gpurun_out/$OUT "$@" > gpurun_out/${OUT}_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/${OUT}_ncu.log
