"""N > 1 host logic of the unstructured cell partition on CPU (gloo, world
size 2): the plan libbte executes (bte_plan_umesh) moves every halo value to
the right slot and covers every face neighbour; skipping the exchange fails."""
import socket

import pytest
import torch.multiprocessing as mp

import bte_inputs as bi
from paper_2305_19400_b200 import build, plan_umesh

from umesh_worker import run


@pytest.fixture(scope="module", autouse=True)
def _lib():
    build.build()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("case", ["tri", "quad", "tet"])
@pytest.mark.parametrize("skip", [False, True])
def test_two_rank_umesh_halo_exchange(tmp_path, case, skip):
    out = str(tmp_path / "res.txt")
    mp.spawn(run, args=(2, _port(), case, skip, out), nprocs=2, join=True)
    assert open(out).read() == ("differ" if skip else "equal")


@pytest.mark.parametrize("P", [1, 2, 3, 5])
def test_umesh_plan_invariants(P):
    m = bi.umesh_tet(3, 3, 2, seed=8)
    plans = [plan_umesh(m, P, r) for r in range(P)]
    assert plans[0]["cell0"] == 0 and sum(q["n_own"] for q in plans) == m.ncells
    assert all(plans[r]["cell0"] + plans[r]["n_own"] == plans[r + 1]["cell0"] for r in range(P - 1))
    for r, q in enumerate(plans):
        owners = [next(k for k in range(P) if plans[k]["cell0"] <= c < plans[k]["cell0"] + plans[k]["n_own"])
                  for c in q["halo"]]
        assert owners == sorted(owners) and r not in owners  # grouped by owner, never self
        for pe in q["peers"]:
            mine = q["halo"][pe["recv_off"]:pe["recv_off"] + pe["recv_cnt"]]
            back = next(x for x in plans[pe["peer"]]["peers"] if x["peer"] == r)
            # what the peer sends me is exactly my halo segment of its cells, in order
            assert list(plans[pe["peer"]]["cell0"] + back["send"]) == list(mine)
    if P == 1:
        assert plans[0]["n_halo"] == 0 and plans[0]["peers"] == []
