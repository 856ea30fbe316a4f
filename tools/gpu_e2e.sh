set -u
cd $GRAFT_REPO_ROOT
O=gpurun_out/e2e
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_cg_fused.py tests/test_gpu_config_sizes.py tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 600 -x > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -2 $O/tests.log
python tools/time_e2e_parts.py
for w in 4 8 16; do
 echo "while $w: $(DS_CG_WHILE_STEPS=$w timeout 300 python bench.py --no-sweep --no-cpu --no-powerlaw --no-mg --no-config5 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["e2e"]["value"], d["e2e"]["seconds"], d["roofline"]["frac"])')"
done
