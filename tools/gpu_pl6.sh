set -u
cd $GRAFT_REPO_ROOT
O=gpurun_out/pl6
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
DS_CSR_TILE_CTAS=2 PROFILE=1 FMTS=csr,coo timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none --csv --log-file $O/launches.csv python tools/powerlaw_kernels.py > $O/launches.log 2>&1
DS_CSR_TILE_CTAS=2 PROFILE=1 FMTS=csr timeout 600 ncu --set full --clock-control none --import-source on -k regex:csr_long_rows -c 2 -o $O/prof_long -f python tools/powerlaw_kernels.py > $O/prof_long.log 2>&1
DS_CSR_TILE_CTAS=2 PROFILE=1 FMTS=csr timeout 600 ncu --set full --clock-control none --import-source on -k regex:csr_tile_kernel -s 1 -c 1 -o $O/prof_tile -f python tools/powerlaw_kernels.py > $O/prof_tile.log 2>&1
ls $O
