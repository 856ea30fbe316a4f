set -u
cd $GRAFT_REPO_ROOT
DS_NATIVE_LIB=$GRAFT_REPO_ROOT/tools/bin/var/libX.so timeout 900 python -m pytest tests/test_gpu_cg_fused.py tests/test_gpu_config_sizes.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
for rep in 1 2; do
  for v in A X; do
    echo "$v bench: $(DS_NATIVE_LIB=$GRAFT_REPO_ROOT/tools/bin/var/lib$v.so timeout 300 python bench.py --no-cpu --no-sweep --no-powerlaw --no-mg 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); f=d["format_switching_192"]; print(d["value"], d["ms_per_step"], d["e2e"]["value"], f["cg_ms_per_step"], f["cg_gflops"])')"
  done
done
