set -u
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in 0 1 2 3 4 5; do
  echo "cfg=$c: $(DS_COO_CFG=$c FMT=coo timeout 120 python tools/tune_spmv.py 2>&1 | tail -1 | cut -c1-160)"
done
