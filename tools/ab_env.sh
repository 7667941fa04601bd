# A/B of environment settings on one workload: tools/ab_env.sh WORKLOAD "EXTRA ARGS" "ENV1" "ENV2" ...
wl=$1; shift; extra=$1; shift
for e in "$@"; do
  for rep in 1 2; do
    env $e python bench.py --workload $wl $extra --steps 5 --warmup 3 --extras none --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl [$e]', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), round(d['e2e']['value']))"
  done
done
