#!/bin/bash
# CSR SpMV tile-shape sweep at 104^3 (DS_CSR_T rows/tile, DS_CSR_S stages,
# DS_CSR_CTAS per SM) + the paired 8-lane kernel for comparison.
cd ${GRAFT_REPO_ROOT:-/root/repo}
DS_CSR_G8=1 FMT=csr timeout 120 python tools/tune_spmv.py 2>&1 | tail -1
for cfg in ${CFGS:-"256 2 1" "128 2 2" "128 3 1" "128 4 1" "192 2 1" "64 3 3" "64 2 4"}; do
  set -- $(echo $cfg | tr ',' ' ')
  DS_CSR_T=$1 DS_CSR_S=$2 DS_CSR_CTAS=$3 FMT=csr timeout 120 python tools/tune_spmv.py 2>&1 | tail -1
done
