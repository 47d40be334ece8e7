"""libbte's NCCL transports between real processes (one GPU each): slab halo
send/recv with and without the overlapped schedule, the band partition's
AllGather, the unstructured partition's pack + send/recv, and the
all-gathered bte_get_energy -- bit-exact against one context, within the
north_star tolerance of the oracle, and broken by the skip-exchange mutation
(S:L429).  NCCL refuses two ranks on one device ("Duplicate GPU detected"),
so this needs >= 2 GPUs and skips otherwise; the same data paths run on one
GPU through the in-process groups (test_gpu_parity.py, test_gpu_umesh.py)."""
import json
import socket

import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module", autouse=True)
def _need_two_gpus():
    import torch
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs (NCCL allows one rank per device)")
    from paper_2305_19400_b200 import build
    build.build()


@pytest.mark.parametrize("kind", ["slab", "overlap0", "band", "umesh"])
@pytest.mark.parametrize("skip", [False, True])
def test_nccl_two_ranks(tmp_path, kind, skip):
    import torch.multiprocessing as mp

    from nccl_worker import run
    out = str(tmp_path / "res.json")
    mp.spawn(run, args=(2, _port(), kind, skip, out), nprocs=2, join=True)
    res = json.load(open(out))
    if skip:
        assert not res["bit_exact"], res
        return
    assert res["bit_exact"], res
    assert res["rel_I_oracle"] <= 1e-10 and res["dT_oracle"] <= 1e-8, res
    assert res["T_same_on_parts"] and res["energy_same_on_ranks"], res
    assert res["energy_rel_vs_oracle"] < 1e-12, res
