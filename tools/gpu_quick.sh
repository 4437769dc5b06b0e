#!/bin/bash
# Quick GPU iteration (run under gpurun): GPU tests, a short bench line
# summary, optionally an ncu capture of one kernel.
#   tools/gpu_quick.sh TAG [kernel-regex-to-profile] [bench args...]
TAG=$1; K=$2; shift 2
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gputests.log 2>&1
echo "tests $?: $(tail -1 gpurun_out/${TAG}_gputests.log)"
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 30 "$@" > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench $?"
python - "$TAG" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/{sys.argv[1]}_bench.json").read().strip().splitlines()[-1])
print(round(d["value"]), d["config"]["workload"], d["config"].get("kernel_path"),
      {k: round(v["ms"], 3) for k, v in d["roofline"]["kernels"].items()})
PY
tail -2 gpurun_out/${TAG}_bench.err
if [ -n "$K" ]; then timeout 300 tools/prof_kernel.sh "$K" ${TAG}_prof "$@" > /dev/null 2>&1; echo "prof $?"; fi
