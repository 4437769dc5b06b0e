#!/bin/bash
# One gpurun call: GPU tests, then the default bench line and the reference arm.
#   gpurun --timeout 1800 -- tools/gpu_check.sh [TAG]
TAG=${1:-check}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gputests.log 2>&1
echo "gpu tests exit $?"
tail -3 gpurun_out/${TAG}_gputests.log
python bench.py ${BENCH_ARGS:-} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench exit $?"
tail -c 600 gpurun_out/${TAG}_bench.json
if [ -z "$NO_REF" ]; then
  python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
  echo "ref exit $?"
fi
