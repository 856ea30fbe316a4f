# conversion profiling at 192^3: wall times, launch lists (CSR->DIA, DIA->CSR,
# COO->CSR) and full ncu captures of the census / fill kernels
set -u
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/conv
NX=192 timeout 300 python tools/time_convert.py
for p in "csr dia" "dia csr" "coo csr" "csr coo"; do
  set -- $p
  SRC=$1 DST=$2 NX=192 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/conv/launch_$1_$2.csv python tools/one_convert.py > /dev/null 2>&1
done
SRC=csr DST=dia NX=192 timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"csr_census_tiles|csr_dia_fill_tiles" -c 2 -o gpurun_out/conv/census_fill -f python tools/one_convert.py > /dev/null 2>&1
SRC=dia DST=csr NX=192 timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"dia_group" -c 2 -o gpurun_out/conv/dia_csr -f python tools/one_convert.py > /dev/null 2>&1
ls -la gpurun_out/conv
