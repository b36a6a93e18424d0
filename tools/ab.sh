#!/bin/bash
# A/B kernel timing of variant libraries, alternating on one box.
# usage: tools/ab.sh <rounds> <config> <family> <variant names...>
R=$1; CFG=$2; FAM=$3; shift 3
for i in $(seq 1 $R); do
  for v in "$@"; do
    MHB_LIB=tools/variants/$v.so timeout 300 python bench.py --config $CFG --family $FAM --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', '$CFG', '$FAM', round(r['kernel_ms'],4), round(r['achieved']/1e3,3), round(r['frac'],4))"
  done
done
