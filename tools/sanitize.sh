#!/bin/bash
# compute-sanitizer over the GPU parity tests (run under gpurun): memcheck on
# every kernel family (parity, CSR/COO pipelines, fused CG, HPCG), racecheck
# and synccheck on the shared-memory pipelines.
cd ${GRAFT_REPO_ROOT:-/root/repo}
mkdir -p gpurun_out
compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py \
    tests/test_gpu_csr_pipe.py tests/test_gpu_coo_pipe.py tests/test_gpu_cg_fused.py \
    tests/test_gpu_hpcg.py tests/test_gpu_convert_paths.py tests/test_gpu_convert_direct.py \
    tests/test_gpu_sort.py -q -x \
    -k "not hashes" > gpurun_out/memcheck.txt 2>&1
# racecheck / synccheck: the solver's device WHILE-loop graph (a conditional
# node) is replaced by chunked graph replays (DS_CG_WHILE_STEPS=0): under these
# two tools the conditional-node solve faults inside the tool (memcheck runs it)
export DS_CG_WHILE_STEPS=0
compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_csr_pipe.py \
    tests/test_gpu_coo_pipe.py tests/test_gpu_parity.py -q -x \
    -k "pipe or tiles or descriptor or spmv_and_spmv_add or long_rows or signed_zeros" \
    > gpurun_out/racecheck.txt 2>&1
compute-sanitizer --tool racecheck --print-limit 20 python -m pytest \
    tests/test_gpu_convert_paths.py tests/test_gpu_convert_direct.py tests/test_gpu_sort.py -q -x \
    > gpurun_out/racecheck_convert.txt 2>&1
compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_csr_pipe.py \
    tests/test_gpu_coo_pipe.py tests/test_gpu_cg_fused.py -q -x > gpurun_out/synccheck.txt 2>&1
tail -n 3 gpurun_out/memcheck.txt gpurun_out/racecheck.txt gpurun_out/racecheck_convert.txt \
    gpurun_out/synccheck.txt
