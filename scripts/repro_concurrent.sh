#!/bin/bash
# Concurrent contexts on shard-sized bands (scripts/shard_pipeline_projection.py) under several
# settings, each in its own process; the tail of each log.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() { local name=$1; shift; echo "== $name"; env "$@" timeout 300 python scripts/shard_pipeline_projection.py > gpurun_out/rc_$name.log 2>&1; echo "rc=$?"; grep -E "^G=|Error|error" gpurun_out/rc_$name.log | sort | uniq | head -8; }
run g2c4a PROJ_G=2 PROJ_C=4
run g2c4b PROJ_G=2 PROJ_C=4
run g2c3 PROJ_G=2 PROJ_C=3
run g2c4blk PROJ_G=2 PROJ_C=4 CUDA_LAUNCH_BLOCKING=1
run g2c4chk PROJ_G=2 PROJ_C=4 DWC_LIB=paper_1608_05179_b200/libdwc_checked.so
run g8 PROJ_G=8 PROJ_C=2,4,6,8
run g4 PROJ_G=4 PROJ_C=2,4,6
