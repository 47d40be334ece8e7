"""Worker for the world-size-2 gloo test of the unstructured cell partition
(N > 1 host logic).  Each rank takes libbte's plan (bte_plan_umesh, the lists
the library executes with NCCL), packs the values of the cells its peers hold
as halo copies, exchanges them over torch.distributed/gloo and checks that
every halo slot then holds the value of the canonical cell the plan names,
and that the owned cells plus the halo cover every face neighbour."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def field(c):
    return np.sin(0.37 * np.asarray(c, dtype=np.float64)) + 2.0


def run(rank, world, port, case, skip_exchange, result_path):
    import torch
    import torch.distributed as dist

    import bte_inputs as bi
    from paper_2305_19400_b200 import plan_umesh

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    mesh = {"tri": bi.umesh_tri(7, 5, 7e-6, 5e-6, seed=3), "quad": bi.umesh_quad(6, 5, 6e-6, 5e-6, seed=4, shuffle=True),
            "tet": bi.umesh_tet(3, 3, 3, seed=5)}[case]
    plan = plan_umesh(mesh, world, rank)
    c0, n_own = plan["cell0"], plan["n_own"]
    own = field(np.arange(c0, c0 + n_own))
    halo = np.zeros(plan["n_halo"])
    if not skip_exchange:
        reqs, bufs = [], []
        for pe in plan["peers"]:
            send = torch.from_numpy(own[pe["send"]].copy())
            recv = torch.zeros(pe["recv_cnt"], dtype=torch.float64)
            bufs.append((pe, recv))
            if send.numel():
                reqs.append(dist.isend(send, pe["peer"]))
            if recv.numel():
                reqs.append(dist.irecv(recv, pe["peer"]))
        for r in reqs:
            r.wait()
        for pe, recv in bufs:
            halo[pe["recv_off"]:pe["recv_off"] + pe["recv_cnt"]] = recv.numpy()
    ok = bool(np.array_equal(halo, field(plan["halo"])))
    # coverage: face neighbours of owned cells are owned or in the halo
    K = mesh.cells.shape[1]
    faces = {}
    for c, cv in enumerate(mesh.cells.tolist()):
        for k in range(K):
            key = (frozenset((cv[(k + 1) % K], cv[(k + 2) % K])) if mesh.dim == 2
                   else frozenset(cv[:k] + cv[k + 1:]))
            faces.setdefault(key, []).append(c)
    need = set()
    for cs in faces.values():
        if len(cs) == 2:
            a, b = cs
            for x, y in ((a, b), (b, a)):
                if c0 <= x < c0 + n_own and not (c0 <= y < c0 + n_own):
                    need.add(y)
    ok = ok and need == set(plan["halo"].tolist())
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([n_own]))
    ok = ok and int(sum(int(t) for t in sizes)) == mesh.ncells
    flags = [torch.zeros(1) for _ in range(world)]
    dist.all_gather(flags, torch.tensor([1.0 if ok else 0.0]))
    if rank == 0:
        with open(result_path, "w") as f:
            f.write("equal" if all(float(t) == 1.0 for t in flags) else "differ")
    dist.destroy_process_group()
