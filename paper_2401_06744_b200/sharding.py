"""Multi-GPU: frames are independent problems, so a batch shards by frame with
no collective on the data path.  One process per GPU; frame f
belongs to rank f mod G.  The only communication is the gather of per-frame
reports (and, on request, of the reconstructed fields) after the solves.

``torch.distributed`` is plumbing (NCCL on the GPU box, gloo in CPU tests)."""

from __future__ import annotations

import numpy as np


def frames_of_rank(n_frames: int, rank: int, world: int) -> list:
    """Global indices of the frames rank `rank` decodes (f mod world == rank)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    return list(range(rank, n_frames, world))


def solve_frames_sharded(masks, known, cfg=None, spacing: float = 1.0, *, solver=None,
                         gather_fields: bool = False, group=None):
    """Decode the frames this rank owns; gather reports on every rank.

    masks (F,H,W), known (F,C,H,W) are the WHOLE batch on every rank (or only
    this rank's rows filled in -- other rows are never read).  Returns
    (fields, reports, owned): fields is (F,C,H,W) with every frame when
    gather_fields else only the owned rows filled, reports[f] is the list of
    per-channel reports of frame f for all F frames.
    """
    import torch.distributed as dist

    if solver is None:
        from .pipelines import solve_frames as solver
    masks = np.asarray(masks)
    known = np.asarray(known, dtype=np.float64)
    if known.ndim == 3:
        known = known[:, None]
    n = masks.shape[0]
    live = dist.is_available() and dist.is_initialized()
    rank = dist.get_rank(group) if live else 0
    world = dist.get_world_size(group) if live else 1
    owned = frames_of_rank(n, rank, world)
    fields = np.zeros_like(known)
    local_reports = {}
    if owned:
        out, reps, _ = solver(masks[owned], known[owned], cfg, spacing)
        for j, f in enumerate(owned):
            fields[f] = out[j]
            local_reports[f] = reps[j]
    if not live or world == 1:
        return fields, [local_reports[f] for f in range(n)], owned
    bucket = [None] * world
    payload = (local_reports, {f: fields[f] for f in owned} if gather_fields else None)
    dist.all_gather_object(bucket, payload, group=group)
    reports = [None] * n
    for reps, flds in bucket:
        for f, r in reps.items():
            reports[f] = r
        if flds:
            for f, a in flds.items():
                fields[f] = a
    return fields, reports, owned
