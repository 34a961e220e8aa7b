for cfgn in cfg2 cfg5; do
for t in "768 384" "896 448"; do
  set -- $t
  DWC_GS_G4=$1 DWC_GS_G2=$2 timeout 900 python bench.py --config $cfgn --steps 2 --warmup 3 --no-cpu-baseline --no-cvf 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$cfgn g4>=$1 g2>=$2', round(d['value'],1), round(d['stage_ms']['gs'],2))"
done; done
