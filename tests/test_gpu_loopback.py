"""libbte's multi-rank code path on ONE GPU through the in-process loopback
transport (include/bte.h, bte_run.nccl_id = "BTELOOP..."): the ranks are
threads of this process, each with its own context and stream; every
send/recv/AllGather the library issues through its NCCL shim is matched
across the ranks at group end and executed as stream-ordered device copies.
So the slab halo exchange (with and without the boundary-plane overlap on the
comm stream), the band partition's in-place AllGather, the unstructured
partition's pack + send/recv + scatter and the all-gathered bte_get_energy run
exactly as under NCCL -- same plans, buffers, kernels, streams and events; only
the wire differs.  Checked bit-exact against one context, within the
north_star tolerance of the oracle, and broken by the skip-exchange mutation
(S:L429).  No kernel waits on another rank (the host rendezvous does)."""
import os
import threading

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _run_threads(world, kind, skip):
    import torch

    import oracle
    from nccl_worker import _case, rank_job, verdict
    from paper_2305_19400_b200 import loopback_unique_id

    p = _case(kind)
    o = oracle.Oracle(p)
    I, T = o.random_state()
    uid = loopback_unique_id()
    res, errs = [None] * world, []

    def job(r):
        try:
            torch.cuda.set_device(0)
            res[r] = rank_job(p, I, T, r, world, kind, skip, uid, 0, stream=torch.cuda.Stream(device=0))
        except Exception as e:  # noqa: BLE001 -- reported below
            errs.append(f"rank {r}: {e!r}")

    old = os.environ.get("BTE_OVERLAP")
    if kind == "overlap0":
        os.environ["BTE_OVERLAP"] = "0"
    try:
        th = [threading.Thread(target=job, args=(r,)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=600)
    finally:
        if kind == "overlap0":
            if old is None:
                os.environ.pop("BTE_OVERLAP", None)
            else:
                os.environ["BTE_OVERLAP"] = old
    assert not errs, errs
    assert all(r is not None for r in res), "a rank did not finish"
    return verdict(p, o, I, T, res, kind)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kind", ["slab", "overlap0", "band", "umesh"])
def test_loopback_ranks(kind, world):
    res = _run_threads(world, kind, skip=False)
    assert res["bit_exact"], res
    assert res["rel_I_oracle"] <= 1e-10 and res["dT_oracle"] <= 1e-8, res
    assert res["T_same_on_parts"] and res["energy_same_on_ranks"], res
    assert res["energy_rel_vs_oracle"] < 1e-12, res


@pytest.mark.parametrize("kind", ["semi", "sctau", "partial"])
def test_loopback_step_variants(kind):
    """The NCCL-path slab exchange under the other integrators / wall kinds:
    semi-implicit step (R-l), self-consistent tau (R-k), partially specular walls (R-i)."""
    res = _run_threads(2, kind, skip=False)
    assert res["bit_exact"], res
    assert res["rel_I_oracle"] <= 1e-10 and res["dT_oracle"] <= 1e-8, res
    assert res["energy_same_on_ranks"], res


@pytest.mark.parametrize("kind", ["slab", "band", "umesh"])
def test_loopback_skip_exchange_mutation(kind):
    """Mutation: without the exchange the parts must disagree with one context."""
    res = _run_threads(2, kind, skip=True)
    assert not res["bit_exact"], res


@pytest.mark.parametrize("kind", ["slab", "overlap0", "band", "umesh"])
def test_loopback_per_rank_timers(kind):
    """The per-rank phase timers bench.py reports at N > 1 (sweep, Newton,
    boundary, halo), observed on the multi-rank path: every rank records its
    halo / AllGather spans (> 0 ms) next to its sweep and Newton, one sweep
    launch set and one Newton per step, nothing truncated."""
    import torch

    from nccl_worker import _case
    from paper_2305_19400_b200 import Solver, loopback_unique_id

    p = _case(kind)
    uid = loopback_unique_id()
    world, nsteps = 2, 6
    res, errs = [None] * world, []

    def job(r):
        try:
            torch.cuda.set_device(0)
            decomp = "band" if kind == "band" else "slab"
            with Solver.from_problem(p, device=0, stream=torch.cuda.Stream(device=0), rank=r, nranks=world,
                                     nccl_id=uid, decomp=decomp) as sv:
                sv.step(2)
                sv.timing_enable(True, 64)
                sv.step(nsteps)
                res[r] = sv.timing_read()
        except Exception as e:  # noqa: BLE001
            errs.append(f"rank {r}: {e!r}")

    old = os.environ.get("BTE_OVERLAP")
    if kind == "overlap0":
        os.environ["BTE_OVERLAP"] = "0"
    try:
        th = [threading.Thread(target=job, args=(r,)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=600)
    finally:
        if kind == "overlap0":
            if old is None:
                os.environ.pop("BTE_OVERLAP", None)
            else:
                os.environ["BTE_OVERLAP"] = old
    assert not errs, errs
    for t in res:
        assert t is not None and t["steps"] == nsteps, t
        assert t["truncated"] == 0, t
        assert t["halo_ms"] > 0.0 and t["sweep_ms"] > 0.0 and t["newton_ms"] > 0.0, t
        assert t["newton_launches"] >= nsteps and t["sweep_launches"] >= nsteps, t  # band: partial + Newton
