set -u
cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-pl5}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_csr_pipe.py tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 600 -x > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -3 $O/tests.log
for cfg in ${SWEEP:-"2" "3" "2 SER" "3 SER"}; do
  set -- $cfg
  b=$1; shift
  E="DS_CSR_TILE_CTAS=$b"
  for f in "$@"; do [ $f = NA ] && E="$E DS_CSR_TILE_NA=1"; [ $f = SER ] && E="$E DS_CSR_SERIAL_LONG=1"; done
  echo "$cfg: $(env $E FMTS=csr timeout 300 python tools/powerlaw_kernels.py 2>&1 | tail -1)" >> $O/sweep.txt
done
cat $O/sweep.txt
