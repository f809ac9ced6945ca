"""Host logic of the multi-GPU path on CPU (gloo, world size 2 and 3): the NCCL
unique-id bootstrap through torch.distributed and the z-slab partition used by
bench.py and the library's slab check."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _uid_worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2107_14790_b200.tgv import broadcast_unique_id
    uid = broadcast_unique_id()
    open(os.path.join(outdir, f"uid{rank}"), "wb").write(uid)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_unique_id_broadcast(tmp_path, world):
    mp.spawn(_uid_worker, args=(world, _port(), str(tmp_path)), nprocs=world, join=True)
    ids = [open(os.path.join(tmp_path, f"uid{r}"), "rb").read() for r in range(world)]
    assert len(ids[0]) == 128 and any(ids[0])
    assert all(i == ids[0] for i in ids)


@pytest.mark.parametrize("nz,world", [(256, 1), (256, 2), (256, 8), (1024, 8), (31, 4), (5, 5)])
def test_slabs_tile_the_grid(nz, world):
    from paper_2107_14790_b200.tgv import slab
    cuts = [slab(nz, r, world) for r in range(world)]
    assert cuts[0][0] == 0 and cuts[-1][1] == nz
    assert all(cuts[r][1] == cuts[r + 1][0] for r in range(world - 1))
    sizes = [b - a for a, b in cuts]
    assert min(sizes) >= 1 and max(sizes) - min(sizes) <= 1
