# same-box A/B of environment switches on the C2 bench line: ENVS="A=1 B=1 ..." ('-' = none)
for rep in 1 2 3; do for e in $ENVS; do
  [ "$e" = "-" ] && ev="" || ev="$e"
  r=$(env $ev timeout 300 python bench.py --no-sub --no-cpu-baseline --steps 30 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); ph=d['phases_ms_per_step']; print('%.4f' % d['ms_per_step'], ' '.join('%s=%.1f' % (k, 1000*v) for k, v in ph.items() if v))")
  echo "rep$rep $e $r"
done; done
