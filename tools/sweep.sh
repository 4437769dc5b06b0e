#!/bin/bash
# Bench a list of flag sets back to back, two rounds (run under gpurun):
#   tools/sweep.sh "--chunk-envs 4096" "--chunk-envs 8192" ...
for r in 1 2; do
  for args in "$@"; do
    out=$(timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 40 $args 2>/dev/null | tail -1)
    echo "round $r [$args] $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), {k: round(x["ms"], 3) for k, x in d["roofline"]["kernels"].items()})')"
  done
done
