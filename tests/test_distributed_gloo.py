"""World-size-2 gloo tests of the shift sharding on CPU.

The per-rank solver is the CPU oracle (tests may call it); the sharding,
broadcast and all-gather logic under test is the package's own."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, golden


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_solver(chf, shifts, nb, batch_size, rtol):
    import sys
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    A = chf.Ahat.cpu().numpy() if isinstance(chf.Ahat, torch.Tensor) else chf.Ahat
    B = chf.Bhat.cpu().numpy() if isinstance(chf.Bhat, torch.Tensor) else chf.Bhat
    C = chf.Chat.cpu().numpy() if isinstance(chf.Chat, torch.Tensor) else chf.Chat
    G, fail = O.tf_eval(A, B, C, shifts, nb=nb, rtol=rtol, threads=1)
    return G, {int(l): int(f) for l, f in enumerate(fail) if f >= 0}


def _worker(rank, world, port, case, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1708_06290_b200 import ControllerHessForm
        from paper_1708_06290_b200.distributed import broadcast_chf, eval_transfer_function_sharded
        F = np.load(os.path.join(ROOT, "tests", "golden", case))
        src = None
        if rank == 0:
            src = ControllerHessForm(Ahat=F["Ahat"], Bhat=F["Bhat"], Chat=F["Chat"],
                                     m=F["Bhat"].shape[1], n=F["Ahat"].shape[0],
                                     p=F["Chat"].shape[0])
        chf = broadcast_chf(src, torch.device("cpu"))
        res = eval_transfer_function_sharded(chf, F["shifts"], nb=8, on_singular="mark",
                                             solver=_oracle_solver)
        np.save(os.path.join(out_dir, f"G{rank}.npy"), res.G.numpy())
        np.save(os.path.join(out_dir, f"f{rank}.npy"),
                np.asarray(sorted(res.failures.items()), dtype=np.int64).reshape(-1, 2))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_transfer_function_gloo(tmp_path, world):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, "failure.npz", str(tmp_path)), nprocs=world, join=True)
    F = golden("failure.npz")
    Gs = [np.load(tmp_path / f"G{r}.npy") for r in range(world)]
    fs = [np.load(tmp_path / f"f{r}.npy") for r in range(world)]
    for r in range(1, world):
        assert np.array_equal(Gs[r], Gs[0], equal_nan=True)
        assert np.array_equal(fs[r], fs[0])
    # failure at global shift 7 (lives on rank 0 of 2), reported on every rank
    assert fs[0].tolist() == [[7, 0]]
    ok = ~np.isnan(F["G"])
    assert np.abs(Gs[0][ok] - F["G"][ok]).max() <= 1e-12 * np.abs(F["G"][ok]).max()
    assert np.isnan(Gs[0][:, 14:16]).all()


def test_shard_bounds():
    from paper_1708_06290_b200.distributed import shard_bounds
    for total in (0, 1, 7, 1000, 4001):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
