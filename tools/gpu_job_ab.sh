# same-box A/B of libmtk variants (abtest/libmtk_<v>.so) on the C2 bench line
for rep in 1 2; do for v in $VARIANTS; do
  r=$(MTK_LIB_PATH=abtest/libmtk_$v.so timeout 300 python bench.py --no-sub --no-cpu-baseline --steps 30 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); ph=d['phases_ms_per_step']; print('%.4f' % d['ms_per_step'], ' '.join('%s=%.1f' % (k, 1000*v) for k, v in ph.items() if v))")
  echo "$v: $r"
done; done
