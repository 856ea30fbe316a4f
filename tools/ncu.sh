#!/bin/bash
# Run on the GPU box (gpurun).  Launch list of every kernel + one full ncu
# capture per hot kernel of tools/profile_kernels.py into gpurun_out/.
set -u
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
NCU=${NCU:-ncu}
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $OUT/launches.csv python tools/profile_kernels.py > $OUT/launches.log 2>&1
for k in ${KERNELS:-dia_pipe csr_pipe coo_pipe cg_update_direction_fused}; do
  $NCU --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o $OUT/prof_$k -f python tools/profile_kernels.py > $OUT/prof_$k.log 2>&1
done
ls -la $OUT
