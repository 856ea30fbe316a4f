set -u
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2f
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_convert_paths.py tests/test_gpu_parity.py tests/test_gpu_sort.py tests/test_matrix_market.py -q -p no:cacheprovider --timeout 300 -x > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
NX=192 timeout 300 python tools/time_convert.py > $O/conv192.json 2>&1
DS_DIA_ONEPASS=0 NX=192 timeout 300 python tools/time_convert.py > $O/conv192_twopass.json 2>&1
NX=104 timeout 300 python tools/time_convert.py > $O/conv104.json 2>&1
FMTS=csr timeout 300 python tools/powerlaw_kernels.py > $O/pl.json 2>&1
DS_SORT_NO_SEGMENTED=1 FMTS=csr timeout 300 python tools/powerlaw_kernels.py > $O/pl_radix.json 2>&1
NX=192 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/conv192_launches.csv python tools/time_convert.py > $O/conv_launches.log 2>&1
PROFILE=1 FMTS=csr timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/pl_launches.csv python tools/powerlaw_kernels.py > $O/pl_launches.log 2>&1
