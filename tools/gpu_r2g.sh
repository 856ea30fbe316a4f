set -u
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2g
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_convert_paths.py tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 300 -x > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
NX=192 timeout 300 python tools/time_convert.py > $O/conv192.json 2>&1
NX=192 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/conv192_launches.csv python tools/time_convert.py > $O/conv_launches.log 2>&1
