set -u
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for w in ${WS:-8 16 32 64}; do
  for rep in 1 2; do
    echo "while $w: $(DS_CG_WHILE_STEPS=$w timeout 300 python bench.py --no-sweep --no-cpu --no-powerlaw --no-mg --no-config5 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["e2e"]["seconds"])')"
  done
done
