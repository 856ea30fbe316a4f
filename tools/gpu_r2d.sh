set -u
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2d
mkdir -p $O
timeout 600 python tools/dbg_rank104.py > $O/dbg_rank.log 2>&1
for w in 0 1 2 4; do echo "== while steps $w" >> $O/e2e.log; DS_CG_WHILE_STEPS=$w NO_PROFILE=1 timeout 300 python tools/time_e2e.py >> $O/e2e.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cg_fused.py tests/test_gpu_csr_pipe.py tests/test_gpu_config_sizes.py -q -p no:cacheprovider --timeout 300 -k "cg or CG" > $O/cgtests.log 2>&1; echo "rc=$?" >> $O/cgtests.log
