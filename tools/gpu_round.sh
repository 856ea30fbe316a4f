#!/bin/bash
# One gpurun call: GPU tests, smoke, bench (both arms), the ncu launch list of
# the bench command and full captures of the hot kernels into gpurun_out/.
set -u
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
( time timeout 600 python bench.py ${BENCH_ARGS:-} > $OUT/bench.json 2> $OUT/bench.err ) 2> $OUT/bench.time
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
if [ -z "${NO_NCU:-}" ]; then
  # launch list of the bench command itself (short run, no CPU leg; the plan
  # fixed to the local DIA the tuner picks outside the profiler -- under ncu
  # its serialised timings can pick another format)
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file $OUT/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu --fixed-plan \
      > $OUT/launches.log 2>&1
  # full captures: "regex skip" pairs over tools/profile_kernels.py (3 SpMVs per
  # format, then eager CG steps: the 4th dia_pipe launch is the CG's fused one)
  for ks in ${KERNELS:-"dia_pipe 3" "csr_pipe 1" "coo_pipe 1" "cg_update_direction_fused 1"}; do
    set -- $ks
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 \
        -o $OUT/prof_$1 -f python tools/profile_kernels.py > $OUT/prof_$1.log 2>&1
  done
fi
ls -la $OUT
