set -u
cd $GRAFT_REPO_ROOT
O=gpurun_out/pl2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for cfg in "3" "3 NA" "3 SER" "6" "16" "64" "16 NA" "64 NA" "16 SER" "64 SER NA"; do
  set -- $cfg
  b=$1; shift
  E="DS_CSR_TILE_CTAS=$b"
  for f in "$@"; do [ $f = NA ] && E="$E DS_CSR_TILE_NA=1"; [ $f = SER ] && E="$E DS_CSR_SERIAL_LONG=1"; done
  echo "$cfg: $(env $E FMTS=csr timeout 300 python tools/powerlaw_kernels.py 2>&1 | tail -1)" >> $O/sweep.txt
done
cat $O/sweep.txt
