"""N > 1 host logic on CPU (gloo, world size 2): libbte's slab plan executed over
torch.distributed reproduces the single-domain oracle bit-exactly; skipping the
exchange breaks it (mutation).  Plus plan invariants for P = 1..8."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import bte_inputs as bi
from paper_2305_19400_b200 import build, plan_slab

from slab_worker import octant_of, run


@pytest.fixture(scope="module", autouse=True)
def _lib():
    build.build()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("case", ["3d", "2d"])
@pytest.mark.parametrize("skip", [False, True])
def test_two_rank_slabs_match_single_domain(tmp_path, case, skip):
    out = str(tmp_path / "res.txt")
    mp.spawn(run, args=(2, _port(), case, 6, skip, out), nprocs=2, join=True)
    res = open(out).read()
    assert res == ("differ" if skip else "equal"), res


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_plan_invariants(P):
    p = bi.config3(n=8)
    p.mesh = bi.Mesh(3, 5, 4, 13, 1e-6, 1e-6, 1e-6)
    plans = [plan_slab(p.mesh, p.dirs, p.bands.nb, P, r) for r in range(P)]
    # owned planes tile [0, nz) in rank order, sizes differ by at most one
    edges = [(q["m0"], q["m0"] + q["n_local"]) for q in plans]
    assert edges[0][0] == 0 and edges[-1][1] == 13
    assert all(edges[i][1] == edges[i + 1][0] for i in range(P - 1))
    sizes = [q["n_local"] for q in plans]
    assert max(sizes) - min(sizes) <= 1
    # every send has exactly one matching receive
    sends = {(r, m["peer"], m["octant"], m["plane"]) for r, q in enumerate(plans) for m in q["msgs"] if m["send"]}
    recvs = {(m["peer"], r, m["octant"], m["plane"]) for r, q in enumerate(plans) for m in q["msgs"] if not m["send"]}
    assert sends == recvs
    # 4 octants up + 4 down per interface; counts = plane cells * 50 dirs * 40 channels
    assert len(sends) == 8 * (P - 1)
    oc = octant_of(p.dirs.s)
    for q in plans:
        for m in q["msgs"]:
            assert m["count"] == 5 * 4 * int((oc == m["octant"]).sum()) * 40
            up = not (m["octant"] & 1)
            if m["send"]:
                assert m["plane"] == (q["m0"] + q["n_local"] - 1 if up else q["m0"])


def test_plan_errors_and_odd_blocks():
    from paper_2305_19400_b200 import BteError
    p = bi.config3(n=8)
    p.mesh = bi.Mesh(3, 5, 4, 3, 1e-6, 1e-6, 1e-6)
    with pytest.raises(BteError):
        plan_slab(p.mesh, p.dirs, p.bands.nb, 4, 3)  # more ranks than planes: rank 3 owns none
    with pytest.raises(BteError):
        plan_slab(p.mesh, p.dirs, p.bands.nb, 2, 2)  # rank out of range
    # odd (cell, octant) blocks: messages carry the even device stride
    d = bi.directions_inplane(12)  # 3 directions per quadrant
    m2 = bi.Mesh(2, 5, 6, 1, 1e-6, 1e-6, 1.0)
    q = plan_slab(m2, d, 5, 2, 0)  # 3 x 5 = 15 doubles -> stride 16
    assert q["axis"] == 1 and all(msg["count"] == 5 * 16 for msg in q["msgs"])
