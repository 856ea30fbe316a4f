# full check: build, GPU tests, smoke, bench (both arms) -> gpurun_out/$TAG
set -u
cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-full}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
tail -2 $O/smoke.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > $O/clocks.csv 2>&1 &
SMI=$!
( time timeout 900 python bench.py > $O/bench.json 2> $O/bench.err ) 2> $O/bench.time
kill $SMI
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
tail -3 $O/bench.err
if [ -n "${NCU:-}" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file $O/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu --fixed-plan > $O/launches.log 2>&1
  for ks in "dia_pipe 3" "csr_pipe 1" "coo_pipe 1" "cg_update_direction_fused 1"; do
    set -- $ks
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 \
        -o $O/prof_$1 -f python tools/profile_kernels.py > $O/prof_$1.log 2>&1
  done
  NX=192 timeout 300 python tools/time_convert.py > $O/convert_192.json 2>&1
  NX=104 timeout 300 python tools/time_convert.py > $O/convert_104.json 2>&1
  for p in "csr dia" "dia csr" "coo csr" "csr coo" "coo dia" "dia dia"; do
    set -- $p
    SRC=$1 DST=$2 NX=192 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file $O/conv_launch_$1_$2.csv python tools/one_convert.py > /dev/null 2>&1
  done
  SRC=csr DST=dia NX=192 timeout 600 ncu --set full --clock-control none --import-source on \
      -k regex:"dia_fill_(rows|csr)" -c 1 -o $O/prof_conv_fill -f python tools/one_convert.py > /dev/null 2>&1
  SRC=dia DST=csr NX=192 timeout 600 ncu --set full --clock-control none --import-source on \
      -k regex:"dia_group" -c 2 -o $O/prof_conv_dia -f python tools/one_convert.py > /dev/null 2>&1
  PROFILE=1 FMTS=csr,coo timeout 600 ncu --set full --clock-control none --import-source on -k regex:"csr_tile_kernel|coo_warp_segments" -s 2 -c 2 \
      -o $O/prof_powerlaw -f python tools/powerlaw_kernels.py > $O/prof_powerlaw.log 2>&1
fi
ls $O
