set -u
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2e
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_config_sizes.py tests/test_gpu_multirank.py tests/test_gpu_dist.py -q -p no:cacheprovider --timeout 450 -x > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 300 python tools/powerlaw_kernels.py > $O/pl.json 2>&1
for c in 4 8 12; do DS_CSR_TILE_CTAS=$c FMTS=csr timeout 300 python tools/powerlaw_kernels.py > $O/pl_c$c.json 2>&1; done
PROFILE=1 FMTS=csr timeout 600 ncu --set full --clock-control none --import-source on -k regex:csr_tile_kernel -s 1 -c 1 -o $O/prof_csr_tile -f python tools/powerlaw_kernels.py > $O/prof_csr_tile.log 2>&1
timeout 300 python tools/time_e2e.py > $O/e2e.log 2>&1
