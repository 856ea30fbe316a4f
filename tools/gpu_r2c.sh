set -u
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_config_sizes.py -k "rank_cg" -x -q -p no:cacheprovider --timeout 300 > $O/rank104.log 2>&1; echo "rc=$?" >> $O/rank104.log
timeout 900 python -m pytest tests/test_gpu_sort.py tests/test_gpu_parity.py tests/test_gpu_convert_paths.py tests/test_gpu_csr_pipe.py -x -q -p no:cacheprovider > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 300 python tools/powerlaw_kernels.py > $O/pl_tiles.json 2> $O/pl_tiles.err
DS_CSR_TILES=0 timeout 300 python tools/powerlaw_kernels.py > $O/pl_binned.json 2> $O/pl_binned.err
for c in 2 3 8; do DS_CSR_TILE_CTAS=$c FMTS=csr timeout 300 python tools/powerlaw_kernels.py > $O/pl_tiles_c$c.json 2>&1; done
PROFILE=1 FMTS=csr timeout 600 ncu --set full --clock-control none --import-source on -k regex:csr_tile_kernel -s 1 -c 1 -o $O/prof_csr_tile -f python tools/powerlaw_kernels.py > $O/prof_csr_tile.log 2>&1
PROFILE=1 FMTS=coo timeout 600 ncu --set full --clock-control none --import-source on -k regex:coo_warp_segments -s 1 -c 1 -o $O/prof_coo_warp -f python tools/powerlaw_kernels.py > $O/prof_coo_warp.log 2>&1
PROFILE=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum --clock-control none --csv --log-file $O/pl_launches.csv python tools/powerlaw_kernels.py > $O/pl_launches.log 2>&1
