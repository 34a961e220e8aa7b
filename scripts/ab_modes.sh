#!/bin/bash
# A/B of library builds (LIBS env) on the linear and cubic cfg3 bands: value and GS ms
for i in 1 2; do
 for mode in "" "--order 3"; do
  for lib in $LIBS; do
   DWC_LIB=$PWD/paper_1608_05179_b200/$lib timeout 300 python bench.py $mode --steps 5 --warmup 3 --no-cpu-baseline --no-cvf 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib [$mode]', round(d['value'],1), round(d['stage_ms']['gs'],2))"
  done
 done
done
