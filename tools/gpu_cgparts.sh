set -u
cd $GRAFT_REPO_ROOT
O=gpurun_out/cgparts
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_cg_fused.py tests/test_gpu_config_sizes.py} -q -p no:cacheprovider --timeout 600 -x > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -3 $O/tests.log
for v in ${VARS:-0 4}; do
  echo "tail variant $v: $(DS_CG_TAIL=$v PERSIST=1 timeout 300 python tools/time_cg_parts.py 2>/dev/null)" >> $O/parts.txt
done
for v in ${VARS:-0 4}; do
  echo "bench variant $v: $(DS_CG_TAIL=$v timeout 300 python bench.py --no-sweep --no-cpu --no-powerlaw --no-mg --no-config5 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["e2e"]["value"], d["roofline"]["frac"])')" >> $O/parts.txt
done
cat $O/parts.txt
