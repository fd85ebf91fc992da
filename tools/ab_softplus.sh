for rep in 1 2; do
for v in default spmufu dspmufu both; do
  if [ $v = default ]; then unset IDEQ_LIB; else export IDEQ_LIB=$PWD/paper_2605_19705_b200/lib/variants/libideq_$v.so; fi
  r=$(timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-tol-run 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])")
  echo "$v $r"
done; done
unset IDEQ_LIB
