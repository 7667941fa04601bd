# e2e vs device-resident C3 time under environment settings: tools/e2e_env.sh DOCS "ENV1" "ENV2" ...
docs=$1; shift
for e in "$@"; do
  env $e python tools/e2e_c3_trace.py $docs 2>&1 | grep -E "^e2e|^device" | tr '\n' ' ' | sed "s/^/[$e] /"; echo
done
