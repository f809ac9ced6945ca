"""Multi-GPU z-slabs across processes, one rank per GPU:
N ranks with tgv_create(nranks = N) over NCCL, in peer halo mode (the fused kernel stores
its boundary planes into the neighbours' halo planes over NVLink) and with the NCCL
send/recv exchange (TGV_PEER_HALO=0), for both schedules and TV-L1: u, v, p, q of every
slab bitwise equal to one context on one GPU, and the energy equal.  Needs >= 2 visible
GPUs (skipped otherwise: the build box and the round-end box have one; the same plans
are pinned on CPU by tests/test_slab_gloo.py and across processes on one GPU by
tests/test_gpu_peer_ipc.py)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir, peer, schedule, model):
    import torch
    import torch.distributed as dist

    import synth
    from paper_2107_14790_b200 import Solver
    from paper_2107_14790_b200.tgv import slab
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["TGV_PEER_HALO"] = "1" if peer else "0"
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    shape = (70, 45, 13 * world + 3)
    h = synth.random_histograms(shape, 21)
    c = [-0.875 + 0.25 * b for b in range(8)]
    z0, z1 = slab(shape[2], rank, world)
    d = Solver.distributed(shape, c, z0, z1, rank).set_schedule(schedule).set_model(model)
    d.load(np.ascontiguousarray(h[z0:z1])).iterate(17)
    one = Solver(shape, c, device=rank).set_schedule(schedule).set_model(model).load(h).iterate(17)
    ok = {}
    for f in ("u", "v", "p", "q"):
        a, b = d.get(f), one.get(f)
        b = b[z0:z1] if f == "u" else b[:, z0:z1]
        ok[f] = bool(np.array_equal(a, b))
    e1, e2 = d.energy(), one.energy()
    ok["E"] = abs(e1["E"] - e2["E"]) <= 1e-12 * abs(e2["E"])
    ok["peer"] = bool(d.info().get("peer_halo")) == peer
    np.save(os.path.join(outdir, f"ok{rank}.npy"), np.array([ok[k] for k in sorted(ok)]))
    dist.barrier()
    d.close()
    one.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("peer,schedule,model", [(True, "fused", "tgv"), (False, "fused", "tgv"),
                                                 (False, "split", "tgv"), (False, "fused", "tvl1")])
def test_ranks_equal_one_gpu_bitwise(tmp_path, world, peer, schedule, model):
    if _ngpus() < world:
        pytest.skip(f"needs {world} GPUs, {_ngpus()} visible")
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(world, _port(), str(tmp_path), peer, schedule, model), nprocs=world, join=True)
    for r in range(world):
        assert np.load(os.path.join(tmp_path, f"ok{r}.npy")).all(), r
