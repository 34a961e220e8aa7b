#!/bin/bash
# A/B of residual-GS build variants on the cfg3 band (GS ms): default lib, then libdwc_<v>.so variants
cd $GRAFT_REPO_ROOT
for lib in "" $@; do
  if [ -z "$lib" ]; then L=paper_1608_05179_b200/libdwc.so; else L=paper_1608_05179_b200/libdwc_$lib.so; fi
  echo "== lib ${lib:-default}"
  DWC_LIB=$L timeout 300 python scripts/rgs_profile.py cfg3 2>&1 | grep -E "band|alone|sum" | head -5
done
