"""Band (channel) partition host logic on CPU (gloo, world size 2; SURVEY 8(f)
f1): oracle sweeps on the channel bands libbte's bte_plan_band assigns, one
all-gather of the per-cell reductions, then the full-channel temperature
update, reproduce the single-domain oracle bit-exactly; skipping the gather
breaks it (mutation).  Plus bte_plan_band invariants and errors."""
import socket

import pytest
import torch.multiprocessing as mp

from paper_2305_19400_b200 import BteError, build, plan_band

from band_worker import run


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
def test_two_rank_bands_match_single_domain(tmp_path, case, skip):
    out = str(tmp_path / "res.txt")
    mp.spawn(run, args=(2, _port(), case, 5, skip, out), nprocs=2, join=True)
    res = open(out).read()
    assert res == ("differ" if skip else "equal"), res


@pytest.mark.parametrize("nb", [1, 2, 5, 40, 55])
def test_plan_band_invariants(nb):
    for P in range(1, min(nb, 9) + 1):
        ranges = [plan_band(nb, P, r) for r in range(P)]
        assert ranges[0][0] == 0 and ranges[-1][1] == nb
        for (a0, a1), (c0, c1) in zip(ranges, ranges[1:]):
            assert a1 == c0
        sizes = [b1 - b0 for b0, b1 in ranges]
        assert min(sizes) >= 1 and max(sizes) - min(sizes) <= 1


def test_plan_band_errors():
    for args in [(4, 5, 0), (4, 0, 0), (4, 2, 2), (4, 2, -1), (0, 1, 0)]:
        with pytest.raises(BteError):
            plan_band(*args)
