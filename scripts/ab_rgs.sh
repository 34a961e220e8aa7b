#!/bin/bash
# A/B of residual-GS build variants on the cfg3 band (GS ms): default lib, then libdwc_<v>.so variants
cd $GRAFT_REPO_ROOT
for lib in "" $@; do
  for psm in 1; do
    if [ -z "$lib" ]; then L=paper_1608_05179_b200/libdwc.so; else L=paper_1608_05179_b200/libdwc_$lib.so; fi
    echo "== lib ${lib:-default} per_sm $psm"
    DWC_LIB=$L DWC_RGS_PER_SM=$psm timeout 120 python scripts/rgs_profile.py cfg3 2>&1 | grep -E "band|alone" | head -2
  done
done
