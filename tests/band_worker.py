"""Worker for the world-size-2 gloo test of the band (channel) partition
("the coupling of the bands only occurs in the
temperature update, which in turn only requires a reduction of intensity
across bands").  Each rank runs the ORACLE sweep on the channels libbte's
bte_plan_band assigns it, reduces them, and the ranks all-gather the per-cell
reductions over torch.distributed/gloo; every rank then runs the oracle's
temperature update over all channels.  Rank 0 checks that T and the union of
the channel slices equal the single-domain oracle run bit-for-bit, and that
every rank holds the same T."""
import dataclasses
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(rank, world, port, case, nsteps, skip_exchange, result_path):
    import torch
    import torch.distributed as dist

    import bte_inputs as bi
    import oracle
    from paper_2305_19400_b200 import plan_band
    from slab_worker import make_case

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    p = make_case(case)
    m = p.mesh
    nb = p.bands.nb
    b0, b1 = plan_band(nb, world, rank)
    mine = np.arange(b0, b1)
    pb = dataclasses.replace(p, bands=bi.subset_bands(p.bands, mine))
    ob = oracle.Oracle(pb, nthreads=1)        # this rank's channels
    of = oracle.Oracle(p, nthreads=1)         # all channels: the temperature update
    T = bi.random_temperature(m, p.seed, p.T_init, 20.0)
    noise = bi.intensity_noise_factor(p.seed, m.ncells, p.dirs.nd, nb, 0.05)
    I = (of.equilibrium(T) * noise)[:, :, b0:b1].copy()
    I0c, betac = of.refresh(T)
    for _ in range(nsteps):
        J = ob.sweep(I, I0c[:, b0:b1], betac[:, b0:b1])
        Dmine = ob.reduce(J, I0c[:, b0:b1])
        if skip_exchange:
            D = np.zeros((m.ncells, nb))
            D[:, b0:b1] = Dmine
        else:
            parts = [torch.empty(0)] * world
            dist.all_gather_object(parts, (b0, Dmine))
            parts.sort(key=lambda t: t[0])
            D = np.concatenate([q[1] for q in parts], axis=1)
        T, I0c, betac = of.temperature_update(D, T, I0c, betac)
        I = J
    got = [None] * world
    dist.all_gather_object(got, (b0, I, T))
    if rank == 0:
        Tf = bi.random_temperature(m, p.seed, p.T_init, 20.0)
        If = of.equilibrium(Tf) * noise
        Ir, Tr, _, _ = of.run(If, Tf, nsteps)
        got.sort(key=lambda t: t[0])
        got_I = np.concatenate([q[1] for q in got], axis=2)
        same_T_all = all(np.array_equal(q[2], got[0][2]) for q in got)
        same = bool(np.array_equal(got_I, Ir) and np.array_equal(got[0][2], Tr) and same_T_all)
        with open(result_path, "w") as f:
            f.write("equal" if same else "differ")
    dist.destroy_process_group()
