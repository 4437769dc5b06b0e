#!/bin/bash
# Round-2 evidence (run under gpurun): bench lines, reference arm, launch
# list of the bench command, ncu --set full captures of every kernel kind.
mkdir -p gpurun_out
O=gpurun_out/r02
timeout 900 python bench.py > ${O}_bench.json 2> ${O}_bench.err; echo "bench $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > ${O}_reference_arm.json 2> ${O}_reference_arm.err; echo "ref $?"
timeout 600 python bench.py --lut-dtype f16 --no-cpu-baseline > ${O}_bench_f16.json 2> ${O}_bench_f16.err; echo "f16 $?"
timeout 600 python bench.py --config 3 --steps 30 > ${O}_bench_c3.json 2> ${O}_bench_c3.err; echo "c3 $?"
timeout 900 python bench.py --config 2 --shadows --steps 10 > ${O}_bench_shadows.json 2> ${O}_bench_shadows.err; echo "shadows $?"
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${O}_launches.csv $CMD > ${O}_launches.log 2>&1; echo "launches $?"
PC="python bench.py --envs 4096 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stream_blur|band_shade|env_epilogue" -s 3 -c 3 -o ${O}_full -f $PC > ${O}_full.log 2>&1; echo "full $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"band_shade" -s 1 -c 1 -o ${O}_full_f16 -f $PC --lut-dtype f16 > ${O}_full_f16.log 2>&1; echo "full f16 $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"shadow_tiled|stream_blur" -s 2 -c 2 -o ${O}_full_shadows -f python bench.py --config 2 --shadows --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > ${O}_full_shadows.log 2>&1; echo "full shadows $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stream_blur|band_shade" -s 2 -c 2 -o ${O}_full_c3 -f python bench.py --config 3 --envs 512 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > ${O}_full_c3.log 2>&1; echo "full c3 $?"
