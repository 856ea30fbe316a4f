set -u
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
# cfg index (threads, E, MINB), stages, CTAs/SM, entries per tile
for c in "0 2 6 1024" "0 3 4 1024" "0 3 5 768" "0 4 3 1024" "0 3 6 512" "1 3 2 2048" "2 3 3 1536" "0 3 4 1536"; do
  set -- $c
  echo "cfg=$1 S=$2 ctas=$3 E=$4: $(DS_COO_CFG=$1 DS_COO_S=$2 DS_COO_CTAS=$3 DS_COO_E=$4 FMT=coo timeout 120 python tools/tune_spmv.py 2>&1 | tail -1)"
done
