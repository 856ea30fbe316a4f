# A/B timing of alternate builds (tools/bin/var/lib*.so) on one box
set -u
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
  for v in ${VARS:-A B C}; do
    echo "$v: $(DS_NATIVE_LIB=$GRAFT_REPO_ROOT/tools/bin/var/lib$v.so FMTS=${FMTS:-csr} timeout 300 python tools/powerlaw_kernels.py 2>&1 | tail -1)"
  done
done
