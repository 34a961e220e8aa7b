# A/B of two builds of the library in one GPU session: DWC_LIB selects the .so (bench GS stage ms)
for i in 1 2 3; do
for lib in libdwc_base.so libdwc.so; do
  DWC_LIB=$PWD/paper_1608_05179_b200/$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-cvf 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value'],1), round(d['stage_ms']['gs'],2))"
done; done
