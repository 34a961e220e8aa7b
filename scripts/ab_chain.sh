#!/bin/bash
# A/B of build variants (libdwc_<v>.so) on the cfg3 band GS time and the chain-floor bin alone,
# twice each, interleaved.  Usage: bash scripts/ab_chain.sh v1 v2 ...  (default lib always first)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for round in 1 2; do
  for lib in "" $@; do
    if [ -z "$lib" ]; then L=paper_1608_05179_b200/libdwc.so; else L=paper_1608_05179_b200/libdwc_$lib.so; fi
    DWC_LIB=$L timeout 300 python scripts/ab_chain.py ${CFG:-cfg3} 2>&1 | tail -1
  done
done
