"""Can two ranks share one GPU in an NCCL communicator? (dev probe) -- runs the
libtgv multi-rank path (tgv_create with a unique id, NCCL halo exchange) on a
small grid with both ranks on cuda:0 and compares with one context."""
import os
import numpy as np
import torch
import torch.distributed as dist
import synth
from paper_2107_14790_b200 import Solver
from paper_2107_14790_b200.tgv import slab

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
shape = (40, 30, 26)
h = synth.random_histograms(shape, 5)
C = [-0.875 + 0.25 * b for b in range(8)]
z0, z1 = slab(shape[2], rank, world)
from paper_2107_14790_b200 import tgv
uid = None
if world > 1:
    t = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        t.copy_(torch.frombuffer(bytearray(tgv.tgv_get_unique_id()), dtype=torch.uint8))
    dist.broadcast(t, 0)
    uid = bytes(t.numpy().tobytes())
for sched in ("fused", "split"):
    s = Solver(shape, C, z_begin=z0, z_end=z1, rank=rank, nranks=world, uid=uid, device=0).set_schedule(sched)
    s.load(np.ascontiguousarray(h[z0:z1])).iterate(20)
    u = s.read_u()
    e = s.energy()
    ref = Solver(shape, C).set_schedule(sched).load(h).iterate(20)
    ok = np.array_equal(u, ref.read_u()[z0:z1])
    print(f"rank {rank} {sched}: bitwise={ok} E={e['E']:.6f} ref={ref.energy()['E']:.6f}", flush=True)
    s.close()
dist.destroy_process_group()
