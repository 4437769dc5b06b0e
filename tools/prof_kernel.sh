#!/bin/bash
# ncu --set full capture of one kernel of the bench step (run under gpurun):
#   tools/prof_kernel.sh <regex> <tag> [bench args...]
K=$1; TAG=$2; shift 2
mkdir -p gpurun_out
CMD="python bench.py --envs ${ENVS:-2048} --steps 2 --warmup 3 --no-e2e --no-cpu-baseline $*"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/${TAG}_plain.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:"$K" -s 2 -c 1 -o gpurun_out/$TAG -f $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu exit $?"
tail -3 gpurun_out/${TAG}_ncu.log
