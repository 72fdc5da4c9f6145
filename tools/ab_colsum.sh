for i in 1 2; do
for v in 0 1; do
if [ $v = 1 ]; then export MTK_NO_COLSUM=1; else unset MTK_NO_COLSUM; fi
python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms_per_step']; print('nocolsum=$v', round(d['ms_per_step'],4), {k: round(v*1000,1) for k,v in p.items()})"
done; done
