import os, socket, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests"); sys.path.insert(0, "/root/repo/oracle")
import torch, torch.distributed as dist, numpy as np
from gpu_util import np_, oracle_all, parity_inputs, to_dev
with socket.socket() as s:
    s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import paper_2505_22296_b200 as P
L, H, Hkv, d = 256, 4, 2, 64
q, k, v, R = parity_inputs(21, L, H, Hkv, d)
orc = oracle_all(q, k, v, R)
def run(engine, side_stream, fam):
    P.set_kernel_family(fam)
    rc = P.RankContext()
    layer = P.SequenceParallelAttention(engine, H, Hkv, d, L, rc)
    ctxm = torch.cuda.stream(torch.cuda.Stream()) if side_stream else torch.cuda.stream(torch.cuda.current_stream())
    with ctxm:
        qt, kt, vt = (to_dev(x).requires_grad_(True) for x in (q, k, v))
        out = layer(qt, kt, vt)
        (out.float() * to_dev(R).float()).sum().backward()
    torch.cuda.synchronize()
    errs = {kk: float(np.max(np.abs(np_(g) - orc[kk]))) for kk, g in (("out", out), ("dq", qt.grad), ("dk", kt.grad), ("dv", vt.grad))}
    print(engine, "side" if side_stream else "default", fam, {k: f"{v:.2e}" for k, v in errs.items()}, flush=True)
for fam in ("tcgen05", "mma"):
    for side in (False, True):
        for engine in ("oracle", "ulysses", "oracle"):
            run(engine, side, fam)
dist.destroy_process_group()
