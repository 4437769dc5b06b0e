#!/bin/bash
# Time library variants back to back (run under gpurun):  tools/ab_run.sh base k2b3 ...
# "base" = paper_2411_04776_b200/libtac_b200.so; others = libtac_b200_<name>.so.  Two rounds.
for r in 1 2; do
  for v in "$@"; do
    lib=paper_2411_04776_b200/libtac_b200.so
    [ "$v" != "base" ] && lib=paper_2411_04776_b200/libtac_b200_$v.so
    val=$(TAC_B200_LIB=$lib python bench.py --no-cpu-baseline --no-e2e --steps 60 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['kernel_ms'],3))")
    echo "round $r $v $val"
  done
done
