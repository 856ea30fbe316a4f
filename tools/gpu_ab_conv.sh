set -u
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
  for v in ${VARS:-A H}; do
    echo "$v: $(DS_NATIVE_LIB=$GRAFT_REPO_ROOT/tools/bin/var/lib$v.so NX=${NX:-192} timeout 300 python tools/time_convert.py 2>&1 | tail -1)"
  done
done
