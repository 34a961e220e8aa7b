#!/bin/bash
# One measurement pass on the GPU box: default bench (+ clocks), reference arm, ncu launch
# list of the bench command, ncu --set full of the GS kernel.  Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
lscpu > gpurun_out/lscpu.txt 2>&1
nvidia-smi -q -d CLOCK > gpurun_out/clocks_q.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench_default rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1; echo "bench_reference rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-cvf --no-pipeline"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "ncu_launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:rgs_kernel -s 6 -c 2 -o gpurun_out/gs_full -f $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu_full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:psf_tc_kernel -s 2 -c 1 -o gpurun_out/psf_full -f $CMD > gpurun_out/ncu_psf.log 2>&1; echo "ncu_psf rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:das_kernel -s 2 -c 1 -o gpurun_out/das_full -f $CMD > gpurun_out/ncu_das.log 2>&1; echo "ncu_das rc=$?"
