set -u
cd $GRAFT_REPO_ROOT
O=gpurun_out/conv
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
NX=192 timeout 300 python tools/time_convert.py
NX=104 timeout 300 python tools/time_convert.py
NX=192 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/conv192_launches.csv python tools/time_convert.py > $O/conv_launches.log 2>&1
python tools/launch_summary.py $O/conv192_launches.csv | head -25
