#!/bin/bash
# Pipelined cfg3 bench (value / sequential / e2e) for library variants: name:lib:contexts ...
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for spec in "$@"; do
  n=${spec%%:*}; rest=${spec#*:}; L=${rest%%:*}; c=${rest#*:}
  DWC_LIB=paper_1608_05179_b200/$L timeout 600 python bench.py --no-cvf --no-cpu-baseline --contexts $c > gpurun_out/abl_$n.log 2>&1
  python - "$n" gpurun_out/abl_$n.log <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], "value %.0f ms %.2f | seq %.0f (%.2f ms) | gs %.2f | e2e %.0f | chain %.2f" % (d["value"], d["ms_per_step"], d["sequential"]["value"], d["sequential"]["ms_per_step"], d["stage_ms"]["gs"], d["e2e"]["value"], d["chain_floor_ms"]))
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
