set -u
cd $GRAFT_REPO_ROOT
O=gpurun_out/conv2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for p in "csr dia" "dia csr"; do
  set -- $p
  SRC=$1 DST=$2 NX=192 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/$1_$2.csv python tools/one_convert.py > /dev/null 2>&1
  python tools/compact_launches.py $O/$1_$2.csv | tail -12
done
