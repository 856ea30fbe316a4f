set -u
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2b
timeout 1200 python -m pytest tests/test_gpu_config_sizes.py tests/test_gpu_multirank.py -k "config or nccl or 104" -q -p no:cacheprovider > gpurun_out/r2b/cfg.log 2>&1; echo "rc=$?" >> gpurun_out/r2b/cfg.log
