"""Worker for the world-size-2 gloo test of the slab decomposition (N > 1 host
logic).  Each rank runs the ORACLE on its slab plus halo planes and executes
the halo plan returned by libbte's bte_plan_slab (the same list the library
runs with NCCL) over torch.distributed/gloo.  Rank 0 checks that the union of
the owned slabs equals the single-domain oracle run bit-for-bit."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def octant_of(s):
    return (4 * (s[:, 0] < 0) + 2 * (s[:, 1] < 0) + (s[:, 2] < 0)).astype(int)


def run(rank, world, port, case, nsteps, skip_exchange, result_path):
    import torch
    import torch.distributed as dist

    import bte_inputs as bi
    import oracle
    from paper_2305_19400_b200 import plan_slab

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    p = make_case(case)
    m = p.mesh
    plan = plan_slab(m, p.dirs, p.bands.nb, world, rank)
    ax = plan["axis"]
    n = [m.nx, m.ny, m.nz]
    lo = max(0, plan["m0"] - 1)
    hi = min(n[ax], plan["m0"] + plan["n_local"] + 1)
    box = [(0, m.nx), (0, m.ny), (0, m.nz)]
    box[ax] = (lo, hi)
    sp = bi.subproblem(p, box)
    o = oracle.Oracle(sp, nthreads=1)
    T = bi.random_temperature(m, p.seed, p.T_init, 20.0, box=box)
    I = o.equilibrium(T) * bi.intensity_noise_factor(p.seed, 0, p.dirs.nd, p.bands.nb, 0.05, mesh=m, box=box)
    I0c, betac = o.refresh(T)
    sm = sp.mesh
    shape = (sm.nz, sm.ny, sm.nx, p.dirs.nd, p.bands.nb)
    oct_ = octant_of(p.dirs.s)

    def plane_view(A, gplane):
        A5 = A.reshape(shape)
        k = gplane - lo
        return A5[k] if ax == 2 else A5[:, k]

    for _ in range(nsteps):
        I, T, I0c, betac = o.run(I, T, 1, I0c, betac)
        if skip_exchange:
            continue
        reqs, recvs = [], []
        for msg in plan["msgs"]:
            dsel = np.nonzero(oct_ == msg["octant"])[0]
            if msg["send"]:
                buf = torch.from_numpy(np.ascontiguousarray(plane_view(I, msg["plane"])[..., dsel, :]))
                assert buf.numel() == msg["count"]
                reqs.append(dist.isend(buf, msg["peer"]))
            else:
                buf = torch.empty(msg["count"], dtype=torch.float64)
                reqs.append(dist.irecv(buf, msg["peer"]))
                recvs.append((msg, dsel, buf))
        for r in reqs:
            r.wait()
        for msg, dsel, buf in recvs:
            v = plane_view(I, msg["plane"])
            v[..., dsel, :] = buf.numpy().reshape(v[..., dsel, :].shape)
    # owned part
    k0 = plan["m0"] - lo
    A5 = I.reshape(shape)
    Tm = T.reshape(shape[:3])
    sl = [slice(None)] * 3
    sl[2 - ax] = slice(k0, k0 + plan["n_local"])
    own_I = np.ascontiguousarray(A5[tuple(sl)])
    own_T = np.ascontiguousarray(Tm[tuple(sl)])
    parts = [None] * world
    dist.all_gather_object(parts, (plan["m0"], own_I, own_T))
    if rank == 0:
        Tf = bi.random_temperature(m, p.seed, p.T_init, 20.0)
        of = oracle.Oracle(p, nthreads=1)
        If = of.equilibrium(Tf) * bi.intensity_noise_factor(p.seed, m.ncells, p.dirs.nd, p.bands.nb, 0.05)
        Ir, Tr, _, _ = of.run(If, Tf, nsteps)
        ref_I = Ir.reshape(m.nz, m.ny, m.nx, p.dirs.nd, p.bands.nb)
        ref_T = Tr.reshape(m.nz, m.ny, m.nx)
        parts.sort(key=lambda t: t[0])
        cat_axis = 2 - ax
        got_I = np.concatenate([q[1] for q in parts], axis=cat_axis)
        got_T = np.concatenate([q[2] for q in parts], axis=cat_axis)
        same = bool(np.array_equal(got_I, ref_I) and np.array_equal(got_T, ref_T))
        with open(result_path, "w") as f:
            f.write("equal" if same else "differ")
    dist.destroy_process_group()


def make_case(case):
    import bte_inputs as bi
    if case == "3d":
        b = bi.subset_bands(bi.silicon_bands(29), [0, 17, 33])
        bcs = [bi.WallBC(1), bi.WallBC(2), bi.WallBC(0, None, 305.0), bi.WallBC(1), bi.WallBC(2),
               bi.WallBC(0, None, 302.0)]
        return bi.small_3d(4, 3, 7, bands=b, bcs=bcs)
    # 2-D, slab axis y, hot spot on +y
    p = bi.config2(n=6)
    p.mesh = bi.Mesh(2, 6, 9, 1, 2e-6, 2e-6, 1.0)
    p.bands = bi.subset_bands(bi.silicon_bands(29), [3, 30])
    p.dirs = bi.directions_control_angle(4, 8)
    p.bcs[3] = bi.WallBC(0, bi.hotspot_profile(6, 2e-6, width=4e-6), 300.0)
    return p
