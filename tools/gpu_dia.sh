set -u
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for pf in ${PFS:-0 1 2}; do
  echo "l2pf $pf parts: $(DS_DIA_L2PF=$pf PERSIST=1 timeout 300 python tools/time_cg_parts.py 2>/dev/null)"
  echo "l2pf $pf bench: $(DS_DIA_L2PF=$pf timeout 300 python bench.py --no-cpu --no-powerlaw --no-mg --no-config5 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["spmv_sweep"]["dia"])')"
done
