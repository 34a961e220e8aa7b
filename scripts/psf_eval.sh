# PSF tensor-core kernel: parity tests, ncu time / pipe utilisation, bench stage times
timeout 120 python -m pytest tests -m gpu -x -q -k "psf or dr or e2e" 2>&1 | grep -E "passed|failed|rror" | tail -3
timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:psf_tc -s 1 -c 1 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-cvf 2>/dev/null | python -c "
import csv,sys
for r in csv.reader(l for l in sys.stdin if l.startswith('\"')):
    if len(r) > 3 and r[-3] != 'Metric Name': print(r[-3], r[-1])"
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-cvf 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stage_ms'])"
