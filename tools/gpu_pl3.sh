set -u
cd $GRAFT_REPO_ROOT
O=gpurun_out/pl3
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
QUICK=1 timeout 300 tools/bin/gather_floor > $O/gf_quick.json 2>&1
WINDOW=1 QUICK=1 timeout 300 tools/bin/gather_floor > $O/gf_quick_window.json 2>&1
DS_L2_WINDOW=1 FMTS=csr timeout 300 python tools/powerlaw_kernels.py > $O/pl_window.json 2>&1
QUICK=1 timeout 600 ncu --set full --clock-control none -k regex:kern -s 9 -c 8 -o $O/prof_gf -f tools/bin/gather_floor > $O/prof_gf.log 2>&1
PROFILE=1 FMTS=csr timeout 600 ncu --set full --clock-control none --import-source on -k regex:csr_tile_kernel -s 1 -c 1 \
      -o $O/prof_tile -f python tools/powerlaw_kernels.py > $O/prof_tile.log 2>&1
ls -la $O
