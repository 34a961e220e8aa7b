#!/bin/bash
# A/B of residual-GS library variants on single bins (GS ms alone) and the cfg3 band
cd $GRAFT_REPO_ROOT
for lib in "" $@; do
  if [ -z "$lib" ]; then L=paper_1608_05179_b200/libdwc.so; else L=paper_1608_05179_b200/libdwc_$lib.so; fi
  echo "== lib ${lib:-default}"
  DWC_LIB=$L timeout 300 python scripts/dbg_cfg5.py cfg3:249 cfg3:255 cfg5:600 cfg5:1023 2>&1 | grep -v "^\[rgs"
  DWC_LIB=$L timeout 300 python scripts/rgs_profile.py cfg3 2>&1 | grep "band"
done
