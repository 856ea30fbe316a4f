#!/bin/bash
# ncu --set full of one kernel (regex $1) from tools/tune_spmv.py (FMT=$2) -> gpurun_out/prof_$1
cd ${GRAFT_REPO_ROOT:-/root/repo}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s 2 -c 1 \
    -o gpurun_out/prof_$1 -f env FMT=$2 python tools/tune_spmv.py > gpurun_out/prof_$1.log 2>&1
tail -1 gpurun_out/prof_$1.log
