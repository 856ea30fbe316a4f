#!/bin/bash
for cfg in "256 3 1" "256 4 1" "128 4 2" "128 3 2" "256 2 1" "128 6 1" "64 8 2"; do
  set -- $cfg
  DS_DIA_T=$1 DS_DIA_S=$2 DS_DIA_CTAS=$3 FMT=dia timeout 120 python tools/tune_spmv.py 2>&1 | tail -1
done
FMT=csr timeout 120 python tools/tune_spmv.py 2>&1 | tail -1
FMT=coo timeout 120 python tools/tune_spmv.py 2>&1 | tail -1
