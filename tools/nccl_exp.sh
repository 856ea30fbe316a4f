# experiment: NCCL world 2 on ONE GPU with fake host ids (net transport over loopback)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ncclexp
cat > /tmp/nccl2.py <<'PY'
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
rank = int(os.environ["RANK"])
os.environ["NCCL_HOSTID"] = f"fakehost{rank}"
dist.init_process_group("gloo")
torch.cuda.set_device(0)
from paper_2209_06478_b200 import dist as D
comm, r, w = D.init_comm(torch.device("cuda", 0))
from paper_2209_06478_b200 import _native
lib = _native.load()
x = torch.full((4,), float(rank + 1), dtype=torch.float64, device="cuda")
y = torch.zeros(8, dtype=torch.float64, device="cuda")
_native.check(lib.ds_allgather_f64(x.data_ptr(), y.data_ptr(), 4, comm, torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
print("rank", rank, y.tolist(), flush=True)
PY
NCCL_SOCKET_IFNAME=lo NCCL_DEBUG=WARN timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29611 /tmp/nccl2.py > gpurun_out/ncclexp/out.txt 2>&1
echo "rc=$?" >> gpurun_out/ncclexp/out.txt
