"""Multi-process z-slab decomposition of the scheme on CPU (gloo), world sizes 2
and 4 with even and uneven cuts (reading R12, §6).

Each rank runs the oracle on its slab [zb, ze) of the global grid, exchanging
only the one-plane halos of an exchange plan (every other halo plane is
poisoned with NaN), and the gathered result must equal the monolithic run
BITWISE.  This pins the halo plans the CUDA runtime implements
(paper_2107_14790_b200/csrc/tgv_runtime.cu, plan_split_a/b, plan_fused,
plan_energy; in the runtime's representation ubar travels as (u_k, u_{k-1})):

  SPLIT, before the dual:   ubar bottom plane -> rank r-1;  vbar(3) top plane -> rank r+1
  SPLIT, before the primal: q_xz, q_yz, q_zz bottom -> r-1;  p_z top -> r+1
  FUSED, once per iteration: ubar, vbar(3), q(6) bottom -> r-1;  ubar, vbar(3), p(3) top -> r+1,
                             then the dual is recomputed on the halo planes (p below, q above)
  energy:                   u, q_xz, q_yz, q_zz bottom -> r-1;  v(3), p_z top -> r+1
  TV-L1 (plan_tvl1_a/_b, plan_tvl1_fused, plan_energy_tvl1): ubar down / p_z up (split);
                             ubar down, ubar + p(3) up then p recomputed at the bottom halo (fused);
                             u down, p_z up (energy) -- no v or q ever travels
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth

# SPLIT plan: two exchanges per iteration
PHASE_A = {"down": [("ubar", 0)], "up": [("vbar", 0), ("vbar", 1), ("vbar", 2)]}
PHASE_B = {"down": [("q", 4), ("q", 5), ("q", 2)], "up": [("p", 2)]}
# FUSED plan: one exchange per iteration; the dual is then recomputed on the halo planes
# (p at the bottom halo, q at the top halo), as the single-sweep kernel does
FUSED = {"down": [("ubar", 0), ("vbar", 0), ("vbar", 1), ("vbar", 2)] + [("q", m) for m in range(6)],
         "up": [("ubar", 0), ("vbar", 0), ("vbar", 1), ("vbar", 2), ("p", 0), ("p", 1), ("p", 2)]}
ENERGY = {"down": [("u", 0), ("q", 4), ("q", 5), ("q", 2)], "up": [("v", 0), ("v", 1), ("v", 2), ("p", 2)]}
# NEXT-4 TV-L1 (plan_tvl1_a / _b / _fused): no v, no q on the wire
TVL1_A = {"down": [("ubar", 0)], "up": []}
TVL1_B = {"down": [], "up": [("p", 2)]}
TVL1_FUSED = {"down": [("ubar", 0)], "up": [("ubar", 0), ("p", 0), ("p", 1), ("p", 2)]}
TVL1_ENERGY = {"down": [("u", 0)], "up": [("p", 2)]}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def exchange(o, plan, rank, world):
    nx, ny, _ = o.shape
    reqs, recvs = [], []
    for name, comp in plan["down"]:
        if rank > 0:
            t = torch.from_numpy(o.get_plane(name, comp, o.zb).copy())
            reqs.append(dist.isend(t, rank - 1))
        if rank < world - 1:
            buf = torch.empty((ny, nx), dtype=torch.float64)
            reqs.append(dist.irecv(buf, rank + 1))
            recvs.append((name, comp, o.ze, buf))
    for name, comp in plan["up"]:
        if rank < world - 1:
            t = torch.from_numpy(o.get_plane(name, comp, o.ze - 1).copy())
            reqs.append(dist.isend(t, rank + 1))
        if rank > 0:
            buf = torch.empty((ny, nx), dtype=torch.float64)
            reqs.append(dist.irecv(buf, rank - 1))
            recvs.append((name, comp, o.zb - 1, buf))
    for r in reqs:
        r.wait()
    for name, comp, z, buf in recvs:
        o.set_plane(name, comp, z, buf.numpy())


def poison_halos(o):
    nx, ny, _ = o.shape
    nan = np.full((ny, nx), np.nan)
    for name, ids in oracle.FIELDS.items():
        for comp in range(len(ids)):
            o.set_plane(name, comp, o.zb - 1, nan)
            o.set_plane(name, comp, o.ze, nan)


def _worker(rank, world, port, shape, cuts, iters, outdir, plan="split"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    zb, ze = cuts[rank], cuts[rank + 1]
    h = synth.random_histograms(shape, 3)[zb:ze]
    tv = plan.startswith("tvl1")
    o = oracle.Oracle(shape, zb=zb, ze=ze, model="tvl1" if tv else "tgv").load(h)
    poison_halos(o)
    for _ in range(iters):
        if plan == "tvl1_split":
            exchange(o, TVL1_A, rank, world)
            o.dual()
            exchange(o, TVL1_B, rank, world)
            o.primal()
        elif plan == "tvl1_fused":
            exchange(o, TVL1_FUSED, rank, world)
            o.dual()
            o.dual_halo()
            o.primal()
        elif plan == "split":
            exchange(o, PHASE_A, rank, world)
            o.dual()
            exchange(o, PHASE_B, rank, world)
            o.primal()
        else:
            exchange(o, FUSED, rank, world)
            o.dual()
            o.dual_halo()
            o.primal()
    exchange(o, TVL1_ENERGY if tv else ENERGY, rank, world)
    e = o.energy()
    sums = torch.tensor([e["alpha1"], e["alpha0"], e["data"], e["dual"]], dtype=torch.float64)
    dist.all_reduce(sums)
    vmax = torch.tensor([e["vmax"]], dtype=torch.float64)
    dist.all_reduce(vmax, op=dist.ReduceOp.MAX)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), u=o.u, v=o.get("v"), p=o.get("p"), q=o.get("q"),
             sums=sums.numpy(), vmax=vmax.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("plan", ["split", "fused", "tvl1_split", "tvl1_fused"])
@pytest.mark.parametrize("cuts", [[0, 8, 16], [0, 4, 8, 12, 16], [0, 1, 5, 6, 16]])
def test_slab_equals_monolithic_bitwise(tmp_path, cuts, plan):
    shape, iters = (7, 6, 16), 25
    world = len(cuts) - 1
    mp.spawn(_worker, args=(world, _free_port(), shape, cuts, iters, str(tmp_path), plan), nprocs=world, join=True)
    model = "tvl1" if plan.startswith("tvl1") else "tgv"
    ref = oracle.Oracle(shape, model=model).load(synth.random_histograms(shape, 3)).iterate(iters)
    parts = [np.load(os.path.join(tmp_path, f"r{r}.npz")) for r in range(world)]
    for name in ("u", "v", "p", "q"):
        got = np.concatenate([p[name] for p in parts], axis=-3)
        assert np.array_equal(got, ref.get(name)), name
    e = ref.energy()
    s = parts[0]["sums"]
    for k, key in enumerate(["alpha1", "alpha0", "data", "dual"]):
        assert abs(s[k] - e[key]) <= 1e-12 * max(1.0, abs(e[key])), key
    assert parts[0]["vmax"][0] == e["vmax"]
