#!/bin/bash
# ncu --set full of one kernel launch: prof_one.sh <kernel-regex> <skip> <out-name> [env...]
set -u
K=$1; S=$2; O=$3; shift 3
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --rays 262144"
env "$@" $CMD > gpurun_out/${O}_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/${O}_plain.log; exit 1; }
env "$@" timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $S -c 1 \
    -o gpurun_out/$O $CMD > gpurun_out/${O}_ncu.log 2>&1
echo "$O rc=$?"
