#!/bin/bash
cd /root/repo
FMT=csr timeout 120 python tools/tune_spmv.py 2>&1 | tail -1
for cfg in "2 7168" "3 4608" "2 8192"; do set -- $cfg; DS_CSR_TILES=1 DS_CSR_S=$1 DS_CSR_ECAP=$2 FMT=csr timeout 120 python tools/tune_spmv.py 2>&1 | tail -1; done
DS_CSR_TILES=1 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
