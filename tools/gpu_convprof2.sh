# the CSR-source census: launch lists (CSR->DIA / CSR->CSR) and one full ncu capture
set -u
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/conv2
for p in "csr dia" "csr csr"; do
  set -- $p
  SRC=$1 DST=$2 NX=192 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/conv2/launch_$1_$2.csv python tools/one_convert.py > /dev/null 2>&1
done
SRC=csr DST=dia NX=192 timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"csr_census_quads|dia_fill_csr" -c 3 -o gpurun_out/conv2/census_quads -f python tools/one_convert.py > /dev/null 2>&1
ls gpurun_out/conv2
