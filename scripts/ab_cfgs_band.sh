#!/bin/bash
# A/B of library variants on whole bands (GS ms): cfg3, cfg4 (full grid), cfg5
cd $GRAFT_REPO_ROOT
for lib in "" $@; do
  if [ -z "$lib" ]; then L=paper_1608_05179_b200/libdwc.so; else L=paper_1608_05179_b200/libdwc_$lib.so; fi
  echo "== lib ${lib:-default}"
  for c in cfg3 cfg4 cfg5; do DWC_LIB=$L timeout 600 python scripts/rgs_profile.py $c 2>&1 | grep "band"; done
done
