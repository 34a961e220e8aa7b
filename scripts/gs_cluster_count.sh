#!/bin/bash
# cfg4/cfg5 GS with fewer concurrent clusters (L2 scatter window) -- experiment
mkdir -p gpurun_out
for cfg in cfg4 cfg5; do
 for cl in 0 48 32 24; do
  if [ $cl = 0 ]; then unset DWC_GS_CLUSTERS; else export DWC_GS_CLUSTERS=$cl; fi
  r=$(timeout 300 python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --no-cvf 2>/dev/null | tail -1)
  echo "$cfg cl=$cl $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],2), round(d["stage_ms"]["gs"],1), round(d["roofline"]["frac"],3))')"
 done
done
