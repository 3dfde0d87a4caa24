"""N>1 path on CPU: world_size-2 gloo processes shard a batch of frames by
f mod G, solve their frames (the CPU oracle stands in for the GPU solver, which
needs a device) and gather the reports -- no data-path collective."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2401_06744_b200.sharding import frames_of_rank, solve_frames_sharded

W, H, F, C = 48, 40, 5, 2


def _oracle_solver(masks, known, cfg, spacing):
    outs, reps = [], []
    for m, k in zip(masks, known):
        o, r = oracle.solve_image(m, k, spacing, oracle.MultigridConfig(block_size=16, overlap=2), threads=1)
        outs.append(o)
        reps.append(r)
    return np.stack(outs), reps, 0.0


def _batch():
    ms, ks = zip(*(oracle.seeded_problem(W, H, 0.1, f, C) for f in range(F)))
    return np.stack(ms), np.stack(ks)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    masks, known = _batch()
    fields, reports, owned = solve_frames_sharded(masks, known, None, 1.0, solver=_oracle_solver,
                                                  gather_fields=True)
    q.put((rank, owned, fields, [[r.iterations for r in fr] for fr in reports]))
    dist.barrier()
    dist.destroy_process_group()


def test_frames_of_rank():
    assert frames_of_rank(64, 3, 8) == list(range(3, 64, 8))
    assert frames_of_rank(5, 1, 2) == [1, 3]
    assert frames_of_rank(1, 1, 2) == []
    assert sorted(sum((frames_of_rank(13, r, 4) for r in range(4)), [])) == list(range(13))
    with pytest.raises(ValueError):
        frames_of_rank(4, 2, 2)


def test_two_rank_gloo_sharding_matches_single_process():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    masks, known = _batch()
    ref, ref_reps, _ = _oracle_solver(masks, known, None, 1.0)
    for rank, owned, fields, iters in got:
        assert owned == list(range(rank, F, 2))
        assert np.array_equal(fields, ref)                      # gathered batch == single-process batch
        assert iters == [[r.iterations for r in fr] for fr in ref_reps]


def test_single_process_path():
    masks, known = _batch()
    fields, reports, owned = solve_frames_sharded(masks, known, None, 1.0, solver=_oracle_solver)
    assert owned == list(range(F)) and len(reports) == F
    assert np.array_equal(fields, _oracle_solver(masks, known, None, 1.0)[0])
