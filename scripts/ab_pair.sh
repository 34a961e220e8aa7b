#!/bin/bash
# Pipelined cfg3 bench under several pair-class thresholds (DWC_RGS_PAIR_MAX_SP) and bands in flight
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for cfgv in "default::2" "p1280:1280:2" "p1024:1024:2" "p1280c3:1280:3" "p896:896:2"; do
  n=${cfgv%%:*}; rest=${cfgv#*:}; pm=${rest%%:*}; c=${rest#*:}
  if [ -n "$pm" ]; then export DWC_RGS_PAIR_MAX_SP=$pm; else unset DWC_RGS_PAIR_MAX_SP; fi
  timeout 600 python bench.py --no-cvf --no-cpu-baseline --contexts $c > gpurun_out/pair_$n.log 2>&1
  python - "$n" gpurun_out/pair_$n.log <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], "value %.0f ms %.2f | seq %.0f (%.2f ms) | gs %.2f | e2e %.0f" % (d["value"], d["ms_per_step"], d["sequential"]["value"], d["sequential"]["ms_per_step"], d["stage_ms"]["gs"], d["e2e"]["value"]))
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
