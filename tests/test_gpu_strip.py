"""Strip mode (single frame cut into horizontal strips, SURVEY 8e / BASELINE config 4b) checked on ONE
GPU with virtual ranks: every rank is a thread with its own plan and stream, the exchanges go through
LocalTransport (device-to-device copies).  The strip solve must reproduce the single-plan solve."""

import threading

import numpy as np
import pytest

import oracle
import paper_2401_06744_b200 as bp
from paper_2401_06744_b200 import strip

pytestmark = pytest.mark.gpu


def _run_virtual(nranks, w, h, c, cfg, mask, known):
    group = strip.LocalGroup(nranks)
    out, errs = [None] * nranks, []

    def work(r):
        try:
            s = strip.StripSolver(w, h, c, cfg, group.transport(r))
            u, reps = s.solve(mask, known)
            out[r] = (s.own, u.cpu().numpy(), reps)
            s.close()
        except BaseException as e:
            errs.append(e)
            group.barrier.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("w,h,dens,seed,nranks", [
    (640, 400, 0.02, 3, 2),
    (640, 400, 0.02, 3, 3),
    (512, 700, 0.05, 5, 4),      # clamped last block row, uneven strips
    (1920, 1080, 0.04, 0, 4),
    (3840, 2160, 0.02, 0, 8),    # the 8-GPU layout of BASELINE config 4 at 4K
])
def test_strip_solve_matches_single_plan(w, h, dens, seed, nranks):
    c = 2
    m, k = oracle.seeded_problem(w, h, dens, seed, channels=c)
    cfg = bp.MultigridConfig(block_size=32, overlap=6)
    ref = bp.solve_image(bp.InpaintingProblem(m, k), "mg-oras", cfg)
    parts = _run_virtual(nranks, w, h, c, cfg, m, k)
    full = np.empty_like(ref.fields)
    covered = 0
    for (lo, hi), u, reps in parts:
        full[:, lo:hi] = u
        covered += hi - lo
        # every rank takes the same decisions: V-cycle counts and residuals agree with the single plan
        for rg, rr in zip(reps, ref.reports):
            assert rg.iterations == rr.iterations and rg.fine_smoother_iterations == rr.fine_smoother_iterations
            assert rg.final_rel_residual == pytest.approx(rr.final_rel_residual, rel=1e-9)
    assert covered == h
    # the norms are summed in a different order (per strip, then over ranks): 1e-9, not bit-identical
    np.testing.assert_allclose(full, ref.fields, rtol=0, atol=1e-9)


def test_strip_geometry_and_halo_plan():
    plan = bp.Plan(3840, 2160, 3, 1, bp.MultigridConfig(), use_graphs=False)
    import ctypes as C
    from paper_2401_06744_b200 import _lib
    n = 8
    ranges = []
    for q in range(n):
        r = (C.c_int * 6)()
        _lib.check(_lib.lib().b200p_plan_strip_ranges(plan.handle, q, n, C.byref(r)))
        ranges.append(tuple(r))
    plan.close()
    assert ranges[0][0] == 0 and ranges[-1][1] == 2160
    for a, b in zip(ranges, ranges[1:]):
        assert a[1] == b[0]                      # strips tile the image
        assert b[4] == a[5] - 1                  # the boundary block row is solved on both sides
    for r in ranges:
        own_lo, own_hi, ext_lo, ext_hi, iy_lo, iy_hi = r
        assert own_lo % 26 == 0 and ext_lo % 2 == 0 and ext_lo <= max(0, own_lo - 1) and ext_hi >= min(2160, own_hi + 1)
        assert ext_hi - own_hi <= 34 and own_lo - ext_lo <= 28   # one-block-deep halos
    # what rank 3 receives is exactly what its neighbours send to it
    recv, _ = strip.halo_plan(ranges, 3)
    sends = []
    for q in range(n):
        if q != 3:
            sends += [(q, a, b) for (dst, a, b) in strip.halo_plan(ranges, q)[1] if dst == 3]
    assert sorted(recv) == sorted(sends)
    rows = strip.coarse_rows(ranges, 1080)
    assert rows[0][0] == 0 and rows[-1][1] == 1080 and all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
