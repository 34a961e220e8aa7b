# two builds (default vs GS_PF=0) on cfg2 and cfg5
for cfgn in cfg2 cfg5; do
for lib in libdwc.so libdwc_pf0.so; do
  DWC_LIB=$PWD/paper_1608_05179_b200/$lib timeout 900 python bench.py --config $cfgn --steps 2 --warmup 3 --no-cpu-baseline --no-cvf 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$cfgn $lib', round(d['value'],1), round(d['stage_ms']['gs'],2))"
done; done
