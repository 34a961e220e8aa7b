#!/bin/bash
# The NEXT-row and variant bench lines (one B200): gpurun_out/next_<name>.log
set -u
mkdir -p gpurun_out
run() { local name=$1; shift; timeout 900 python bench.py --no-cpu-baseline "$@" > gpurun_out/next_$name.log 2>&1; echo "$name rc=$?"; }
run cfg3_cubic --order 3
run cfg3_dr --dr
run cfg3_alt --alt
run cfg3_paper --paper
run cfg3_snap --input snapshots
run cfg3_dense_kernel --kernel dense
run cfg4 --config cfg4 --steps 2 --warmup 3 --no-cvf --no-pipeline
run cfg5 --config cfg5 --steps 2 --warmup 3 --no-cvf --no-pipeline
# ncu capture of the residual kernel's cluster mode on cfg4 (full grid): DRAM bytes per launch
CMD4="python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu-baseline --no-cvf"
timeout 900 $CMD4 > gpurun_out/plain4.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:rgs_kernel -s 1 -c 1 -o gpurun_out/rgs_cfg4_full -f $CMD4 > gpurun_out/ncu_cfg4.log 2>&1; echo "ncu_cfg4 rc=$?"
