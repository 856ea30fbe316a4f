# row-slot DIA fill: parity tests + A/B timing (DS_DIA_FILL_ROWS=0/1) -> gpurun_out/$TAG
set -u
cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-fillrows}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest -q -p no:cacheprovider ${TESTS:-tests/test_gpu_convert_paths.py tests/test_gpu_property.py tests/test_gpu_parity.py tests/test_gpu_convert_direct.py tests/test_gpu_config_sizes.py} -m gpu -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
for rep in 1 2; do
  for v in ${VARS:-0 1}; do
    echo "rows=$v 192: $(DS_DIA_FILL_ROWS=$v NX=192 timeout 300 python tools/time_convert.py 2>&1 | tail -1)"
    echo "rows=$v 104: $(DS_DIA_FILL_ROWS=$v NX=104 timeout 300 python tools/time_convert.py 2>&1 | tail -1)"
  done
done > $O/ab.txt
cat $O/ab.txt
for p in ${PAIRS:-csr:dia}; do
  s=${p%:*}; d=${p#*:}
  SRC=$s DST=$d NX=192 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file $O/conv_launch_${s}_${d}.csv python tools/one_convert.py > /dev/null 2>&1
done
if [ -n "${NCUFULL:-}" ]; then
  for m in 1 2; do
    DS_DIA_FILL_ROWS=$m SRC=csr DST=dia NX=192 timeout 600 ncu --set full --clock-control none --import-source on \
        -k regex:"dia_fill_(rows|pipe)" -c 1 -o $O/prof_fill$m -f python tools/one_convert.py > $O/prof_fill$m.log 2>&1
  done
fi
