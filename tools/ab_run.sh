#!/bin/bash
# Time library variants back to back (run under gpurun):  tools/ab_run.sh "bench args" base k2b3 ...
# "base" = paper_2411_04776_b200/libtac_b200.so; others = libtac_b200_<name>.so.  Two rounds.
ARGS=$1; shift
for r in 1 2; do
  for v in "$@"; do
    lib=paper_2411_04776_b200/libtac_b200.so
    [ "$v" != "base" ] && lib=paper_2411_04776_b200/libtac_b200_$v.so
    val=$(TAC_B200_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 40 $ARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), {k: round(x['ms'], 3) for k, x in d['roofline']['kernels'].items()})")
    echo "round $r $v $val"
  done
done
