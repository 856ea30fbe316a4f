#!/bin/bash
# compute-sanitizer over the GPU parity tests (run under gpurun)
cd /root/repo
mkdir -p gpurun_out
compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x \
    -k "not slow and not hashes" > gpurun_out/memcheck.txt 2>&1
compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x \
    -k "spmv_and_spmv_add or long_rows or signed_zeros" > gpurun_out/racecheck.txt 2>&1
tail -3 gpurun_out/memcheck.txt gpurun_out/racecheck.txt
