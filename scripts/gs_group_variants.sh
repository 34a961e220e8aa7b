# CTAs-per-bin thresholds on the linear- and cubic-predictor bands
for t in "768 384" "800 416" "832 448" "864 448" "896 448"; do
  set -- $t
  for mode in "" "--order 3"; do
    DWC_GS_G4=$1 DWC_GS_G2=$2 timeout 300 python bench.py $mode --steps 3 --warmup 3 --no-cpu-baseline --no-cvf 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$mode g4>=$1 g2>=$2', round(d['value'],1), round(d['stage_ms']['gs'],2))"
  done
done
