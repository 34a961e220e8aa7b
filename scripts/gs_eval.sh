mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
DWC_GS_PROFILE=1 N=1170 SWEEPS=1000 timeout 120 python scripts/gs_profile_one.py 2>&1 | grep gs-prof | head -3
timeout 300 python scripts/gs_chain.py cfg3 2>&1 | tail -6
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-cvf > gpurun_out/b3.json 2>gpurun_out/b3.err; python -c "
import json; d=json.load(open('gpurun_out/b3.json')); print(d['value'], d['stage_ms'], d['roofline']['frac'])"
