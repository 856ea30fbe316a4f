# power-law iteration: build, CSR/COO parity tests, timings per CTA count, ncu of the tile kernels
set -u
cd $GRAFT_REPO_ROOT
O=gpurun_out/${TAG:-pl}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_csr_pipe.py tests/test_gpu_coo_pipe.py tests/test_gpu_parity.py} -q -p no:cacheprovider --timeout 600 -x > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for b in ${CTAS:-3}; do
  DS_CSR_TILE_CTAS=$b DS_COO_TILE_CTAS=$b timeout 300 python tools/powerlaw_kernels.py > $O/pl_$b.json 2>&1
done
for k in ${KERNELS:-csr_tile_kernel}; do
  PROFILE=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o $O/prof_$k -f python tools/powerlaw_kernels.py > $O/prof_$k.log 2>&1
done
ls -la $O
