# A/B of an environment switch on the C3 bench: tools/ab_env.sh VAR=VALUE [reps]
kv=$1; reps=${2:-2}
for rep in $(seq $reps); do
  for v in base alt; do
    if [ $v = base ]; then r=$(timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-tol-run 2>/dev/null | tail -1)
    else r=$(env $kv timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-tol-run 2>/dev/null | tail -1); fi
    echo "$v $(echo "$r" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])")"
  done
done
