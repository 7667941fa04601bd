# A/B of library variants on one workload: tools/ab_wl.sh WORKLOAD "EXTRA ARGS" variant...
wl=$1; shift; extra=$1; shift
for v in "$@"; do
  if [ "$v" = "default" ]; then unset BM_LIB_PATH; else export BM_LIB_PATH=tools/_prof/$v.so; fi
  for rep in 1 2; do
    python bench.py --workload $wl $extra --steps 5 --warmup 2 --extras none --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl $v', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), round(d['e2e']['value']))"
  done
done
