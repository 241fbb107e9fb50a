"""Multi-GPU sharding of the shifted solves.

Shifts are independent, so the path shards with exactly two collectives
and none on the data path:

  1. one broadcast of the reduced triple (Ahat, Bhat, Chat) from the rank
     that reduced it (NCCL over NVLink/NVSwitch when the tensors are on GPU);
  2. each rank solves a contiguous slice of the shifts with the single-GPU
     library call;
  3. one all-gather of the G slices (+ the failure map).

One process per GPU, launched by torchrun; ``torch.distributed`` provides the
plumbing (``nccl`` on GPUs, ``gloo`` in the CPU tests).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .errors import SingularShiftError
from .hessenberg import ControllerHessForm


def shard_bounds(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous balanced slice [lo, hi) of ``total`` items for ``rank``."""
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _dev_tensor(a, device) -> torch.Tensor:
    t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.asarray(a))
    return t.to(device)


def broadcast_chf(chf: ControllerHessForm | None, device, src: int = 0,
                  group=None) -> ControllerHessForm:
    """Broadcast the reduced triple from ``src`` to every rank (column-major
    device tensors on ``device``)."""
    rank = dist.get_rank(group)
    dims = torch.zeros(3, dtype=torch.int64, device=device)
    if rank == src:
        dims[:] = torch.tensor([chf.n, chf.m, chf.p])
    dist.broadcast(dims, src, group=group)
    n, m, p = (int(v) for v in dims.tolist())
    out = []
    for name, shape in (("Ahat", (n, n)), ("Bhat", (n, m)), ("Chat", (p, n))):
        rows, cols = shape
        buf = torch.empty((cols, rows), dtype=torch.float64, device=device)  # column-major storage
        if rank == src:
            buf.copy_(_dev_tensor(getattr(chf, name), device).to(torch.float64).t())
        if buf.numel():
            dist.broadcast(buf, src, group=group)
        out.append(buf.t())
    return ControllerHessForm(Ahat=out[0], Bhat=out[1], Chat=out[2], m=m, n=n, p=p)


def gather_slices(G_local: torch.Tensor, fail_local: dict[int, int], lo: int, total: int,
                  m: int, group=None):
    """All-gather per-rank G slices (p x cnt*m complex) into p x total*m, and
    merge the failure maps (local shift index -> global)."""
    world = dist.get_world_size(group)
    device = G_local.device
    p = G_local.shape[0]
    counts = [shard_bounds(total, r, world) for r in range(world)]
    maxcnt = max(hi - lo_ for lo_, hi in counts)
    # (maxcnt*m, p, 2) real view, padded
    send = torch.zeros((maxcnt * m, p, 2), dtype=torch.float64, device=device)
    if G_local.numel():
        send[:G_local.shape[1]] = torch.view_as_real(G_local.t().contiguous())
    recv = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(recv, send, group=group)
    fl = torch.full((maxcnt,), -1, dtype=torch.int64, device=device)
    for l, i in fail_local.items():
        fl[l] = i
    frecv = [torch.empty_like(fl) for _ in range(world)]
    dist.all_gather(frecv, fl, group=group)
    cols, failures = [], {}
    for r, (rlo, rhi) in enumerate(counts):
        cols.append(torch.view_as_complex(recv[r][:(rhi - rlo) * m].contiguous()))
        fr = frecv[r][:rhi - rlo].cpu().numpy()
        for l in np.nonzero(fr >= 0)[0]:
            failures[rlo + int(l)] = int(fr[l])
    G = torch.cat(cols, dim=0).t() if cols else torch.zeros((p, 0), dtype=torch.complex128)
    return G, failures


def eval_transfer_function_sharded(chf: ControllerHessForm, shifts, nb: int = 32,
                                   batch_size: int | None = None, *,
                                   on_singular: str = "raise", singular_rtol=None,
                                   group=None, solver=None):
    """Shift-sharded ``eval_transfer_function`` over all ranks of ``group``:
    rank r solves shifts[lo_r:hi_r]; every rank returns the full (G, failures).

    ``solver(chf, shifts, nb, batch_size, singular_rtol) -> (G, failures)``
    defaults to the single-GPU library call; tests substitute a CPU solver
    to exercise the sharding and gather logic on gloo.
    """
    from .solvers import TransferFunctionResult, eval_transfer_function

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    sh = np.asarray(shifts.cpu() if isinstance(shifts, torch.Tensor) else shifts,
                    dtype=np.complex128).ravel()
    lo, hi = shard_bounds(len(sh), rank, world)
    if solver is None:
        res = eval_transfer_function(chf, sh[lo:hi], nb=nb, batch_size=batch_size,
                                     on_singular="mark", singular_rtol=singular_rtol)
        G_loc, f_loc = res.G, res.failures
    else:
        G_loc, f_loc = solver(chf, sh[lo:hi], nb, batch_size, singular_rtol)
    if isinstance(chf.Ahat, torch.Tensor) and chf.Ahat.is_cuda:
        device = chf.Ahat.device
    else:
        device = torch.device("cpu") if dist.get_backend(group) == "gloo" else torch.device(
            "cuda", torch.cuda.current_device())
    G_loc = _dev_tensor(G_loc, device).to(torch.complex128)
    G, failures = gather_slices(G_loc, f_loc, lo, len(sh), chf.m, group=group)
    if failures and on_singular == "raise":
        raise SingularShiftError(sorted(failures.items()))
    return TransferFunctionResult(G=G, shifts=sh, failures=failures)
