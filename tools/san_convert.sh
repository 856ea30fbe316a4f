# compute-sanitizer racecheck + memcheck over the conversion tests (run under gpurun)
cd ${GRAFT_REPO_ROOT:-/root/repo}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/san
export DS_CG_WHILE_STEPS=0
timeout 1500 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_convert_paths.py tests/test_gpu_convert_direct.py -q -x -p no:cacheprovider > gpurun_out/san/racecheck_convert.txt 2>&1
tail -3 gpurun_out/san/racecheck_convert.txt
timeout 1500 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_convert_paths.py tests/test_gpu_convert_direct.py -q -x -p no:cacheprovider > gpurun_out/san/memcheck_convert.txt 2>&1
tail -3 gpurun_out/san/memcheck_convert.txt
for i in 1 2; do NX=192 python tools/time_convert.py | cut -c1-200; done
