"""The NCCL path of the shift-sharded transfer function (distributed.py:
broadcast of the reduced triple, contiguous shift slice, all-gather of G and
the failure rows) on the one GPU a test box has: a world of one NCCL rank
runs every collective of the N-rank path; results must equal the single-GPU
call bitwise.  (The N-rank slicing / gather logic is covered by the 2-rank
gloo tests in test_distributed_gloo.py.)"""

import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import paper_1708_06290_b200 as ss
from paper_1708_06290_b200.distributed import broadcast_chf, eval_transfer_function_sharded

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_nccl_world_of_one_matches_single_gpu():
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                            device_id=dev)
    try:
        sysb = ss.random_stable_system(300, 10, 4, seed=11, circular=False)
        chf = ss.reduce_controller_hessenberg(sysb.A, sysb.B, sysb.C, block_size=32).to(dev)
        chf_b = broadcast_chf(chf, dev)
        shifts = 1j * np.logspace(-1, 1, 37) * np.sqrt(300)
        ev = np.linalg.eigvals(chf.Ahat.cpu().numpy())
        shifts[5] = ev[0]  # a singular shift: its failure row must come back too
        ref = ss.eval_transfer_function(chf, shifts, nb=64, on_singular="mark")
        res = eval_transfer_function_sharded(chf_b, shifts, nb=64, on_singular="mark")
        G = res.G.cpu().numpy() if isinstance(res.G, torch.Tensor) else res.G
        Gr = ref.G.cpu().numpy() if isinstance(ref.G, torch.Tensor) else ref.G
        assert res.failures == ref.failures
        ok = [l for l in range(len(shifts)) if l not in ref.failures]
        cols = np.concatenate([np.arange(l * 10, (l + 1) * 10) for l in ok])
        assert np.array_equal(G[:, cols], Gr[:, cols])
    finally:
        dist.destroy_process_group()
