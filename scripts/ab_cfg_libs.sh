#!/bin/bash
# A/B of library builds (LIBS env) on several configs (CFGS env): value, GS ms, roofline frac
for cfg in ${CFGS:-cfg3 cfg4 cfg5}; do
 for lib in $LIBS; do
  r=$(DWC_LIB=$PWD/paper_1608_05179_b200/$lib timeout 300 python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --no-cvf 2>/dev/null | tail -1)
  echo "$cfg $lib $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],2), round(d["stage_ms"]["gs"],1), round(d["roofline"]["frac"],3))' 2>&1 | tail -1)"
 done
done
