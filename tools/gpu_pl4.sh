set -u
cd $GRAFT_REPO_ROOT
O=gpurun_out/pl4
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for cfg in "0 3" "1 3" "2 3" "0 2" "1 2" "2 2" "0 4" "1 4"; do
  set -- $cfg
  echo "exp $1 ctas $2 serial: $(DS_CSR_SERIAL_LONG=1 DS_CSR_TILE_EXP=$1 DS_CSR_TILE_CTAS=$2 FMTS=csr timeout 300 python tools/powerlaw_kernels.py 2>&1 | tail -1)" >> $O/sweep.txt
done
cat $O/sweep.txt
