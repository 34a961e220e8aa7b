# GS CTAs-per-bin thresholds (DWC_GS_G4 / DWC_GS_G2 env knobs of gs_group_size): bench GS ms
for t in "896 448" "896 512" "896 576" "896 640"; do
  set -- $t
  DWC_GS_G4=$1 DWC_GS_G2=$2 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-cvf 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('g4>=$1 g2>=$2', round(d['value'],1), round(d['stage_ms']['gs'],2))"
done
