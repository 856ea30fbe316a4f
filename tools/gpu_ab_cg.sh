set -u
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
  for v in ${VARS:-A D}; do
    echo "$v: $(DS_NATIVE_LIB=$GRAFT_REPO_ROOT/tools/bin/var/lib$v.so PERSIST=1 timeout 300 python tools/time_cg_parts.py 2>/dev/null)"
    echo "$v bench: $(DS_NATIVE_LIB=$GRAFT_REPO_ROOT/tools/bin/var/lib$v.so timeout 300 python bench.py --no-cpu --no-sweep --no-powerlaw --no-mg --no-config5 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["e2e"]["value"])')"
  done
done
