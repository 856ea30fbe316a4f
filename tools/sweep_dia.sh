#!/bin/bash
# DIA SpMV tile-shape sweep at 104^3: DS_DIA_T rows/tile, DS_DIA_S stages,
# DS_DIA_CTAS per SM.
cd ${GRAFT_REPO_ROOT:-/root/repo}
FMT=dia timeout 120 python tools/tune_spmv.py 2>&1 | tail -1
for cfg in ${CFGS:-"256 2 1" "128 2 2" "128 3 2" "64 3 4" "128 4 1" "256 3 1"}; do
  set -- $cfg
  DS_DIA_T=$1 DS_DIA_S=$2 DS_DIA_CTAS=$3 FMT=dia timeout 120 python tools/tune_spmv.py 2>&1 | tail -1
done
