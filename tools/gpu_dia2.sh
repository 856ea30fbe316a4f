set -u
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for cfg in "0 3 2" "1 3 2" "1 4 2" "0 4 2" "1 3 3" "1 2 3"; do
  set -- $cfg
  E="DS_DIA_S=$2 DS_DIA_CTAS=$3"; [ $1 = 1 ] && E="$E DS_DIA_GATHER_NA=1"
  echo "na=$1 S=$2 ctas=$3: $(env $E timeout 300 python bench.py --no-cpu --no-powerlaw --no-mg --no-config5 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["spmv_sweep"]["dia"]["ms"])')"
done
