#!/bin/bash
cd /root/repo
POWERLAW=1 FMT=csr timeout 200 python tools/tune_spmv.py 2>&1 | tail -1
DS_NO_L2_WINDOW=1 POWERLAW=1 FMT=csr timeout 200 python tools/tune_spmv.py 2>&1 | tail -1
python -m pytest tests -m gpu -q -x 2>&1 | tail -1
