# the N > 1 bench path on one GPU (DS_BENCH_SAME_GPU=1: all ranks on cuda:0)
set -u
cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-multi}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for N in ${NS:-2 4}; do
  DS_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
     --master-addr 127.0.0.1 --master-port $((29600 + N)) bench.py --gpus $N --steps 20 --warmup 10 \
     ${BARGS:---nx 48} > $O/bench_n$N.json 2> $O/bench_n$N.err
  echo "N=$N rc=$?" >> $O/rc.txt
  DS_BENCH_SAME_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
     --master-addr 127.0.0.1 --master-port $((29700 + N)) bench.py --impl reference --gpus $N --steps 2 --warmup 3 \
     ${BARGS:---nx 48} > $O/bench_ref_n$N.json 2> $O/bench_ref_n$N.err
  echo "ref N=$N rc=$?" >> $O/rc.txt
done
cat $O/rc.txt
