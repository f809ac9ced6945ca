"""Peer halo mode across processes, on one GPU.

Two processes own z-slabs of one grid.  They map each other's state and hand-over
flags with CUDA IPC (tgv_peer_export / tgv_peer_import; the records travel over gloo),
so the fused TGV kernel of each writes its boundary planes into the other's halo planes
and waits on the other's system-scope flag -- the protocol a multi-GPU run uses with
TGV_PEER_HALO=1, minus NVLink.  The slabs are leaf contexts (no NCCL communicator is
needed: NCCL refuses two ranks on one GPU); their initial borders are the neighbour's
initial boundary planes.  The result must equal one context bitwise.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import synth

pytestmark = pytest.mark.gpu
C8 = [-0.875 + 0.25 * b for b in range(8)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shape, cuts, iters, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2107_14790_b200 import Solver, tgv
    z0, z1 = cuts[rank], cuts[rank + 1]
    h = synth.random_histograms(shape, 13)
    s = Solver.leaf(shape, C8, z0, z1).load(np.ascontiguousarray(h[z0:z1]))
    u = s.read_u()
    mine = (u[0].copy(), u[-1].copy(), tgv.tgv_peer_export(s.ctx))
    got = [None] * world
    dist.all_gather_object(got, mine)
    if rank > 0:
        s.set_border(0, u=got[rank - 1][1])
        tgv.tgv_peer_import(s.ctx, 0, got[rank - 1][2])
    if rank + 1 < world:
        s.set_border(1, u=got[rank + 1][0])
        tgv.tgv_peer_import(s.ctx, 1, got[rank + 1][2])
    dist.barrier()
    s.iterate(iters)
    np.save(os.path.join(outdir, f"u{rank}.npy"), s.read_u())
    np.save(os.path.join(outdir, f"p{rank}.npy"), s.get("p"))
    dist.barrier()  # nobody frees its state while a neighbour's kernel may still write into it
    s.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cuts", [[0, 11, 23], [0, 5, 6, 23]])
def test_two_processes_peer_halo_equals_single_context(tmp_path, cuts):
    from paper_2107_14790_b200 import Solver
    shape, iters = (47, 29, 23), 9
    world = len(cuts) - 1
    mp.spawn(_worker, args=(world, _free_port(), shape, cuts, iters, str(tmp_path)), nprocs=world, join=True)
    ref = Solver(shape, C8).load(synth.random_histograms(shape, 13)).iterate(iters)
    u = np.concatenate([np.load(os.path.join(tmp_path, f"u{r}.npy")) for r in range(world)], axis=0)
    p = np.concatenate([np.load(os.path.join(tmp_path, f"p{r}.npy")) for r in range(world)], axis=1)
    assert np.array_equal(u, ref.read_u())
    assert np.array_equal(p, ref.get("p"))
