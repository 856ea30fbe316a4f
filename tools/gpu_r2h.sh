set -u
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2h
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
FMTS=csr timeout 300 python tools/powerlaw_kernels.py > $O/pl.json 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > $O/clocks.csv 2>&1 &
SMI=$!
( time timeout 900 python bench.py > $O/bench.json 2> $O/bench.err ) 2> $O/bench.time
kill $SMI
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
