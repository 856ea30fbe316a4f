# A/B of DIA fill variants (tools/bin/var/lib$V.so) at 192^3 + 104^3; tests on the default build
set -u
cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-fillab}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest -q -p no:cacheprovider ${TESTS:-tests/test_gpu_convert_paths.py tests/test_gpu_property.py tests/test_gpu_parity.py} -m gpu -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -2 $O/pytest.log
for rep in 1 2; do
  for v in ${VARS:-U8}; do
    lib=${v%%:*}; ev=""; [ "$lib" != "$v" ] && ev=${v#*:}
    echo "$v 192: $(env $ev DS_NATIVE_LIB=$GRAFT_REPO_ROOT/tools/bin/var/lib$lib.so NX=192 timeout 300 python tools/time_convert.py 2>&1 | tail -1)"
  done
done > $O/ab.txt
for p in ${PAIRS:-csr:dia}; do
  s=${p%:*}; d=${p#*:}
  SRC=$s DST=$d NX=192 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file $O/conv_launch_${s}_${d}.csv python tools/one_convert.py > /dev/null 2>&1
done
