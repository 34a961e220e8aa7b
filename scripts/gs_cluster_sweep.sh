for n in 0 64 56 48 40; do
  DWC_GS_CLUSTERS=$n timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-cvf 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('clusters=$n', round(d['value'],1), round(d['stage_ms']['gs'],2))"
done
