#!/bin/bash
# ncu evidence for the fused kernel (run under gpurun): launch list + one full capture.
set -x
mkdir -p gpurun_out
CMD="python bench.py --envs ${ENVS:-1024} --steps 3 --warmup 3 --no-e2e --no-cpu-baseline ${EXTRA:-}"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:frame_kernel -s 2 -c 1 -o gpurun_out/${TAG:-prof_fused} -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "exit $?"
