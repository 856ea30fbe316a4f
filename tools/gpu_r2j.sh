set -u
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2j
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 tools/bin/gather_floor > $O/gather_floor.json 2>&1
timeout 300 python tools/powerlaw_kernels.py > $O/pl.json 2>&1
for k in csr_tile_kernel coo_warp_segments; do
  PROFILE=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o $O/prof_$k -f python tools/powerlaw_kernels.py > $O/prof_$k.log 2>&1
done
ls -la $O
