#!/bin/bash
# COO SpMV sweep at 104^3: DS_COO_CFG tile shape (see coo_pipe_launch), plus
# DS_COO_S stages / DS_COO_CTAS per SM overrides; the warp kernel for comparison.
cd ${GRAFT_REPO_ROOT:-/root/repo}
DS_COO_WARP=1 FMT=coo timeout 120 python tools/tune_spmv.py 2>&1 | tail -1
for cfg in ${CFGS:-"0" "1" "2" "3" "4" "5"}; do
  set -- $cfg
  env DS_COO_CFG=$1 ${2:+DS_COO_S=$2} ${3:+DS_COO_CTAS=$3} FMT=coo timeout 120 python tools/tune_spmv.py 2>&1 | tail -1
done
