# same-box A/B of environment switches on the attack line: ENVS="A=1 ..." ('-' = none)
for rep in 1 2 3; do for e in $ENVS; do
  [ "$e" = "-" ] && ev="" || ev="$e"
  r=$(env $ev timeout 300 python bench.py --workload attack --no-cpu-baseline --steps 200 --warmup 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4f ms' % d['ms_per_step'])")
  echo "rep$rep $e $r"
done; done
