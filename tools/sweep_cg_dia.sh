for cfg in "128 3 2" "128 4 2" "256 3 1" "128 2 3" "64 4 4" "128 3 2"; do
  set -- $cfg
  v=$(DS_DIA_T=$1 DS_DIA_S=$2 DS_DIA_CTAS=$3 timeout 300 python bench.py --no-cpu --no-sweep --no-config5 --no-mg --no-powerlaw --steps 2000 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])")
  echo "T=$1 S=$2 CTAS=$3 -> $v"
done
