# A/B of ring-kernel variants on C2 (tools/_prof/*.so built by tools/build_variant.py)
for v in "$@"; do
  if [ "$v" = "default" ]; then unset BM_LIB_PATH; else export BM_LIB_PATH=tools/_prof/$v.so; fi
  for rep in 1 2; do
    python bench.py --workload c2 --steps 10 --warmup 3 --extras none --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), round(d['e2e']['value']))"
  done
done
