set -u
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_coo_pipe.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
for c in "0 2 6 1024" "3 2 8 1024" "4 2 8 768" "5 2 5 1536"; do
  set -- $c
  echo "cfg=$1 S=$2 ctas=$3 E=$4: $(DS_COO_CFG=$1 DS_COO_S=$2 DS_COO_CTAS=$3 DS_COO_E=$4 FMT=coo timeout 120 python tools/tune_spmv.py 2>&1 | tail -1 | cut -c1-150)"
done
