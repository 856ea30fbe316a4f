set -u
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2a
nvidia-smi -q | grep -i -A3 "compute mode\|MIG Mode" > gpurun_out/r2a/smi.txt 2>&1
which nvidia-cuda-mps-control >> gpurun_out/r2a/smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_multirank.py -x -q -p no:cacheprovider > gpurun_out/r2a/dist.log 2>&1; echo "rc=$?" >> gpurun_out/r2a/dist.log
bash tools/nccl_exp.sh
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_multirank.py --deselect tests/test_gpu_dist.py > gpurun_out/r2a/gpu_all.log 2>&1; echo "rc=$?" >> gpurun_out/r2a/gpu_all.log
