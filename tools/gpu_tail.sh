set -u
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in ${VARS:-0 1 2 3}; do
  echo "var $v parts: $(DS_CG_TAIL_VAR=$v PERSIST=1 timeout 300 python tools/time_cg_parts.py 2>/dev/null)"
  echo "var $v bench: $(DS_CG_TAIL_VAR=$v timeout 300 python bench.py --no-sweep --no-cpu --no-powerlaw --no-mg --no-config5 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["e2e"]["value"])')"
done
