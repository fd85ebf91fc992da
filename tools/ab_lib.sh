for rep in 1 2 3; do
for v in new v8; do
  if [ $v = new ]; then unset IDEQ_LIB; else export IDEQ_LIB=$PWD/paper_2605_19705_b200/lib/variants/libideq_v8.so; fi
  r=$(timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-tol-run 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])")
  echo "$v $r"
done; done
