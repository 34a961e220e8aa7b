# A/B of library builds on the DAS stage (bench stage ms): LIBS env
for i in 1 2; do
for lib in $LIBS; do
  DWC_LIB=$PWD/paper_1608_05179_b200/$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-cvf 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['stage_ms']['das'],3), round(d['stage_ms']['psf'],3))"
done; done
