#!/bin/bash
cd /root/repo
for f in csr coo; do FMT=$f timeout 120 python tools/tune_spmv.py 2>&1 | tail -1; done
for f in csr coo; do POWERLAW=1 FMT=$f timeout 200 python tools/tune_spmv.py 2>&1 | tail -1; done
