# same-box A/B of libmtk builds (abtest/libmtk_<v>.so; "cur" = the in-tree build) on the attack line
for rep in 1 2 3; do for v in $VARIANTS; do
  [ "$v" = "cur" ] && lp="" || lp="MTK_LIB_PATH=abtest/libmtk_$v.so"
  r=$(env $lp timeout 300 python bench.py --workload attack --no-cpu-baseline --steps 200 --warmup 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4f ms  e2e %.3g q/s' % (d['ms_per_step'], d['e2e']['value']))")
  echo "rep$rep $v $r"
done; done
