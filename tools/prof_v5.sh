#!/bin/bash
# ncu evidence for the two-kernel path (run under gpurun): the plain run, the
# launch list of the same command, and one --set full capture of each kernel.
set -x
mkdir -p gpurun_out
CMD="python bench.py --envs ${ENVS:-1024} --steps 3 --warmup 3 --no-e2e --no-cpu-baseline ${EXTRA:-}"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"band_|env_epi" -s 3 -c 3 -o gpurun_out/${TAG:-prof_v5} -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "exit $?"
