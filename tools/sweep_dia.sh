#!/bin/bash
cd /root/repo
for f in dia csr coo; do FMT=$f timeout 120 python tools/tune_spmv.py 2>&1 | tail -1; done
DS_COO_V1=1 FMT=coo timeout 120 python tools/tune_spmv.py 2>&1 | tail -1
