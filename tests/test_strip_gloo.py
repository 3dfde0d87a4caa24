"""Strip mode, host side on CPU (no GPU): the strip geometry, the halo plan, and the
torch.distributed transport (gloo, world size 3) against the in-process LocalTransport on the same
data: partial-norm all-reduce, one-block-deep halo rows of the iterate, all-gather of the
restricted residual.  The GPU side (kernels restricted to row ranges, exchange callback) is covered
by tests/test_gpu_strip.py with virtual ranks on one device."""

import os
import socket
import threading

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2401_06744_b200 import strip

H, W, P, WORLD = 700, 24, 2, 3
BLOCK, OVERLAP = 32, 6


def _fields(rank):
    """What a rank holds before an exchange: its own rows carry the rank's signature, the rest junk."""
    g = torch.Generator().manual_seed(100 + rank)
    u = torch.rand((P, H, W), generator=g, dtype=torch.float64) + 10.0 * (rank + 1)
    rc = torch.rand((P, (H + 1) // 2, W // 2), generator=g, dtype=torch.float64) - 5.0 * (rank + 1)
    return u, rc


def _expected(ranges):
    own = [_fields(q) for q in range(len(ranges))]
    h1 = (H + 1) // 2
    rows1 = strip.coarse_rows(ranges, h1)
    exp = []
    for r, rg in enumerate(ranges):
        u, rc = _fields(r)
        for q, a, b in strip.halo_plan(ranges, r)[0]:
            u[:, a:b] = own[q][0][:, a:b]
        for q, (a, b) in enumerate(rows1):
            rc[:, a:b] = own[q][1][:, a:b]
        exp.append((u, rc))
    return exp


def _exercise(t, ranges):
    u, rc = _fields(t.rank)
    rs = torch.tensor([1.0 + t.rank, 0.5 * (t.rank + 1)], dtype=torch.float64)
    fl = torch.tensor([t.rank == 1, 0], dtype=torch.int32)
    t.sum_(rs)
    t.max_(fl)
    t.halo(u, ranges)
    t.gather_rows(rc, strip.coarse_rows(ranges, (H + 1) // 2))
    return u, rc, rs, fl


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ranges = strip.strip_ranges(H, BLOCK, OVERLAP, world)
    u, rc, rs, fl = _exercise(strip.TorchDistTransport(), ranges)
    q.put((rank, u.numpy(), rc.numpy(), rs.numpy(), fl.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_strip_ranges_cover_and_overlap():
    for h, n in ((700, 3), (2160, 8), (4320, 8), (64, 2)):
        rg = strip.strip_ranges(h, BLOCK, OVERLAP, n)
        assert rg[0][0] == 0 and rg[-1][1] == h
        for a, b in zip(rg, rg[1:]):
            assert a[1] == b[0] and b[4] <= a[5]          # strips tile the image; boundary block rows shared
        for own_lo, own_hi, ext_lo, ext_hi, iy_lo, iy_hi in rg:
            assert ext_lo <= own_lo < own_hi <= ext_hi and iy_lo < iy_hi
            assert own_lo % 2 == 0 and ext_lo % 2 == 0
    with pytest.raises(ValueError):
        strip.strip_ranges(8, BLOCK, OVERLAP, 5)              # more ranks than row pairs: an empty strip
    two = strip.strip_ranges(2160, BLOCK, OVERLAP, 8, levels=2)
    assert len(two) == 2 and all(len(lv) == 8 for lv in two)
    assert all(two[1][q][0] == two[0][q][0] // 2 for q in range(8))


def test_local_transport_threads():
    ranges = strip.strip_ranges(H, BLOCK, OVERLAP, WORLD)
    group = strip.LocalGroup(WORLD)
    got = [None] * WORLD

    def work(r):
        got[r] = _exercise(group.transport(r), ranges)

    ts = [threading.Thread(target=work, args=(r,)) for r in range(WORLD)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    exp = _expected(ranges)
    for r in range(WORLD):
        u, rc, rs, fl = got[r]
        assert torch.equal(u, exp[r][0]) and torch.equal(rc, exp[r][1])
        assert rs.tolist() == [6.0, 3.0] and fl.tolist() == [1, 0]


def test_gloo_transport_matches_local():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(WORLD):
        rank, u, rc, rs, fl = q.get(timeout=120)
        res[rank] = (u, rc, rs, fl)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    exp = _expected(strip.strip_ranges(H, BLOCK, OVERLAP, WORLD))
    for r in range(WORLD):
        u, rc, rs, fl = res[r]
        assert np.array_equal(u, exp[r][0].numpy()) and np.array_equal(rc, exp[r][1].numpy())
        assert rs.tolist() == [6.0, 3.0] and fl.tolist() == [1, 0]


@pytest.mark.parametrize("height,nranks,levels", [(700, 3, 1), (2160, 8, 2), (4320, 8, 3), (1080, 2, 2), (333, 4, 1)])
def test_native_halo_plan_matches_the_python_plan(height, nranks, levels):
    """The row intervals the library's NCCL exchange walks (b200p_strip_halo_plan) are those of strip.halo_plan,
    per pair of ranks in the same order on the sending and on the receiving side (NCCL matches the sends and
    receives of a pair in issue order), and together they fill every halo exactly once."""
    rg = strip.strip_ranges(height, BLOCK, OVERLAP, nranks, levels)
    by_level = [rg] if levels == 1 else rg
    for l in range(levels):
        plans = [strip.native_halo_plan(by_level, l, r) for r in range(nranks)]
        for r in range(nranks):
            recv, send = plans[r]
            want_recv, want_send = strip.halo_plan(by_level[l], r)
            assert sorted(recv) == sorted(want_recv) and sorted(send) == sorted(want_send)
            for q in range(nranks):
                if q == r:
                    continue
                # what r sends to q, in order == what q expects from r, in order
                assert [(a, b) for p, a, b in send if p == q] == [(a, b) for p, a, b in plans[q][0] if p == r]
            own_lo, own_hi, ext_lo, ext_hi = by_level[l][r][:4]
            covered = sorted((a, b) for _, a, b in recv)
            halo_rows = (own_lo - ext_lo) + (ext_hi - own_hi)
            assert sum(b - a for a, b in covered) == halo_rows
            assert all(covered[i][1] <= covered[i + 1][0] for i in range(len(covered) - 1))
