"""Debug: dist.RankCG at world 1 (peer / nccl transport, graph / eager) vs the
single-partition engine on growing grids; prints iterations and the first
history entry that differs."""
import json
import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2209_06478_b200 as ds  # noqa: E402
from paper_2209_06478_b200 import dist as D  # noqa: E402

dev = torch.device("cuda", 0)
with socket.socket() as s:
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
out = {}
for nx in [int(v) for v in os.environ.get("GRIDS", "16,32,48,64,104").split(",")]:
    spec = ds.GridSpec(nx, nx, nx)
    part = ds.generate_partition(spec, 0, space=ds.MemorySpace.DEVICE, device=dev)
    split = ds.split_local_remote(ds.PartitionedProblem(spec, [part]), 0)
    ds.convert_inplace(split.local, ds.FormatId.DIA)
    ref = ds.cg(ds.SERIAL, split.local, part.b, tol=1e-9)
    rh = ref.residual_history
    row = {"ref_iters": ref.iterations}
    for transport in ("peer", "nccl"):
        for graph in (True, False):
            eng = D.RankCG(spec, part, split, dev, 1e-9, 500, transport=transport)
            st = torch.cuda.current_stream(dev).cuda_stream
            eng.setup(st)
            if graph:
                eng.capture_step()
            for _ in range(ref.iterations + 8):
                eng.replay() if graph else eng.step(st)
            sc = eng.scalars()
            h = eng.hist[:sc.iter + 1].cpu().numpy()
            k = min(len(h), len(rh))
            diff = np.flatnonzero(np.abs(h[:k] - rh[:k]) > 1e-8 * rh[:k])
            row[f"{transport}_{'graph' if graph else 'eager'}"] = {
                "iters": int(sc.iter), "done": int(sc.done),
                "first_diff": int(diff[0]) if diff.size else None,
                "h_at": [float(v) for v in h[diff[0]:diff[0] + 2]] if diff.size else None}
            eng.close()
    out[nx] = row
    print(json.dumps({nx: row}), flush=True)
dist.destroy_process_group()
