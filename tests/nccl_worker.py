"""Worker of tests/test_gpu_nccl.py: one process per GPU (torchrun-style env
or mp.spawn), libbte's own NCCL transports -- slab halo send/recv (with and
without the boundary-plane overlap), the band partition's AllGather, the
unstructured cell partition's pack + send/recv, and the all-gathered energy --
against one context of the same problem.  Rank 0 writes a JSON verdict."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def _case(kind):
    import bte_inputs as bi
    if kind == "umesh":
        return bi.small_umesh(3, (4, 3, 3), shuffle=True)
    b = bi.subset_bands(bi.silicon_bands(29), [0, 17, 33, 39])
    bcs = [bi.WallBC(1), bi.WallBC(2), bi.WallBC(0, None, 305.0), bi.WallBC(1), bi.WallBC(2),
           bi.WallBC(0, None, 302.0)]
    p = bi.small_3d(6, 5, 9, bands=b, bcs=bcs)
    if kind == "semi":  # semi-implicit step (reading R-l) beyond the explicit dt bound
        p.dt, p.semi = 20.0 * p.dt, 1
    elif kind == "sctau":  # self-consistent tau (reading R-k)
        p.tau_mode = 1
    elif kind == "partial":  # partially specular walls (reading R-i)
        p.bcs = [bi.WallBC(3, None, 300.0, 0.6), bi.WallBC(2), bi.WallBC(0, None, 305.0), bi.WallBC(3, None, 300.0, 0.25),
                 bi.WallBC(1), bi.WallBC(0, None, 302.0)]
    return p


def rank_job(p, I, T, rank, world, kind, skip, nccl_id, device, stream=None, nsteps=5):
    """One rank: its part of the problem through libbte's multi-rank path."""
    from paper_2305_19400_b200 import Solver
    from paper_2305_19400_b200.bte import DEBUG_SKIP_EXCHANGE
    decomp = "band" if kind == "band" else "slab"
    sv = Solver.from_problem(p, device=device, stream=stream, rank=rank, nranks=world, nccl_id=nccl_id, decomp=decomp)
    try:
        if skip:
            sv.set_debug(DEBUG_SKIP_EXCHANGE, 1)
        if kind == "band":
            sv.set_state(np.ascontiguousarray(I[:, :, sv.b0:sv.b1]), T)
        else:
            c0 = sv.cell0 if kind == "umesh" else sv.z0 * (sv.ncells // max(1, sv.nz_local))
            sv.set_state(I[c0:c0 + sv.ncells], T[c0:c0 + sv.ncells])
        E0 = sv.energy()
        sv.step(nsteps)
        E1 = sv.energy()
        return {"rank": rank, "I": sv.intensity(), "T": sv.temperature(), "E0": E0, "E1": E1,
                "b0": sv.b0, "b1": sv.b1}
    finally:
        sv.close()


def verdict(p, o, I, T, allr, kind, nsteps=5) -> dict:
    """The gathered parts against one context (bit-exact) and the oracle (north_star tolerance)."""
    from paper_2305_19400_b200 import Solver
    allr = sorted(allr, key=lambda d: d["rank"])
    if kind == "band":
        Ig = np.concatenate([d["I"] for d in allr], axis=2)
        Tg = allr[0]["T"]
        same_T = all(np.array_equal(d["T"], Tg) for d in allr)
    else:
        Ig = np.concatenate([d["I"] for d in allr])
        Tg = np.concatenate([d["T"] for d in allr])
        same_T = True
    with Solver.from_problem(p, device=0) as s1:
        s1.set_state(I, T)
        s1.step(nsteps)
        I1, T1 = s1.intensity(), s1.temperature()
    Io, To, _, _ = o.run(I, T, nsteps)
    if kind == "band":  # reading R-h: the parts' sums associate differently -> rounding-level agreement
        same = bool(np.max(np.abs(Tg - T1)) <= 1e-10 and np.max(np.abs(Ig / I1 - 1)) <= 1e-12)
    else:
        same = bool(np.array_equal(Ig, I1) and np.array_equal(Tg, T1))
    return {"bit_exact": same,
            "rel_I_oracle": float(np.max(np.abs(Ig - Io) / np.abs(Io))),
            "dT_oracle": float(np.max(np.abs(Tg - To))),
            "T_same_on_parts": bool(same_T),
            "energy_same_on_ranks": len({(d["E0"], d["E1"]) for d in allr}) == 1,
            "energy_rel_vs_oracle": abs(allr[0]["E0"] / o.energy(I) - 1)}


def run(rank, world, port, kind, skip, out):
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2305_19400_b200 import nccl_unique_id

    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    p = _case(kind)
    o = oracle.Oracle(p)
    I, T = o.random_state()
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    if kind == "overlap0":
        os.environ["BTE_OVERLAP"] = "0"
    mine = rank_job(p, I, T, rank, world, kind, skip, obj[0], rank)
    allr = [None] * world
    dist.all_gather_object(allr, mine)
    if rank == 0:
        json.dump(verdict(p, o, I, T, allr, kind), open(out, "w"))
    dist.destroy_process_group()
