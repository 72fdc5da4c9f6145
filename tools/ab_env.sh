# A/B an env toggle on the bench step: bash tools/ab_env.sh VAR
for i in 1 2; do
for v in 0 1; do
if [ $v = 1 ]; then export $1=1; else unset $1; fi
python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms_per_step']; print('$1=$v', round(d['ms_per_step'],4), {k: round(v*1000,1) for k,v in p.items()})"
done; done
