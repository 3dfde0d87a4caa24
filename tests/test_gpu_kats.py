"""Known-answer tests of the REFERENCE's own suite, run on this backend with the reference's inputs and
against outputs the reference wrote (tests/golden/golden_kats.npz, make_golden.py --kats), plus the
identity the block-solve kernels use for the local CG stop test, pinned against a direct r.r."""

import os

import numpy as np
import pytest

import oracle
import paper_2401_06744_b200 as bp

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_kats.npz"))


def test_blocksolver_matches_scalar_local_solve():
    """tests/test_solvers.py:156-169 (TestBlockSolver.test_matches_scalar_local_solve): clamped blocks in
    both axes, bs.solve_blocks(bs.gather(r), target, max_iters=4096) to 1e-12 of the scalar local solves."""
    m, k = oracle.seeded_problem(80, 56, 0.15, 8)
    part = bp.build_partition(80, 56, 32, 6)
    bs = bp.BlockSolver(m, 1.0, part, bp.build_weights(part), alpha=0.5)
    r = np.random.default_rng(12345).normal(size=(56, 80))
    r[m] = 0.0
    assert np.array_equal(r, G["kat_blocks_r"])
    target = 1e-5 * float(np.vdot(r, r))
    assert target == float(G["kat_blocks_target"])
    tiles = bs.gather(r)
    batched = bs.solve_blocks(tiles, target, max_iters=4096)
    np.testing.assert_allclose(batched, G["kat_blocks_v"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(bs.solve_blocks(r, target, max_iters=4096), batched, rtol=0, atol=0)   # gather fused
    bad = tiles.copy()
    bad[1, 0, 0] += 1.0                     # block 1's first column lies inside block 0
    with pytest.raises(ValueError, match="disagree on their overlaps"):
        bs.solve_blocks(bad, target, max_iters=4096)


def test_scatter_weighted_is_the_combine_kernel_alone():
    """solvers.py:307-314 (tests/test_solvers.py:171-180 compares it with extend_add_weighted): the sweeps'
    combine kernel (K2b) on its own, fed the reference's local corrections: bit-for-bit np.bincount order."""
    m, _ = oracle.seeded_problem(80, 56, 0.15, 8)
    part = bp.build_partition(80, 56, 32, 6)
    wts = bp.build_weights(part)
    bs = bp.BlockSolver(m, 1.0, part, wts, alpha=0.5)
    got = bs.scatter_weighted(G["kat_blocks_v"])
    assert np.array_equal(got, G["kat_blocks_scatter"])
    ref = np.zeros((56, 80))
    for i, rect in enumerate(part.rects()):
        bp.extend_add_weighted(ref, rect, wts.block(part, i), G["kat_blocks_v"][i])
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12)
    # a partition of unity: scattering the gather of a field returns the field
    f = np.random.default_rng(5).normal(size=(56, 80))
    np.testing.assert_allclose(bs.scatter_weighted(bs.gather(f)), f, rtol=0, atol=1e-13)


def test_single_level_v_cycle_reduces_to_smoothing():
    """tests/test_multigrid.py:218-233: on a one-level hierarchy v_cycle == nu_pre + nu_post oras_sweeps,
    bit for bit; and both equal the reference's own iterate."""
    m, k = oracle.seeded_problem(32, 32, 0.1, 4)
    prob = bp.InpaintingProblem(m, k)
    cfg = bp.MultigridConfig()
    hier = bp.build_hierarchy(prob, cfg)
    assert len(hier) == 1
    lev = hier.levels[0]
    b = lev.rhs[0]
    u_cycle = prob.flat_init(0)
    bp.v_cycle(hier, 0, u_cycle, b, cfg)
    u_manual = prob.flat_init(0)
    bs = bp.BlockSolver(m, 1.0, lev.part, lev.weights, cfg.solver.alpha)
    bp.oras_sweeps(lev.op, bs, b, u_manual, max_sweeps=cfg.nu_pre + cfg.nu_post, stop_norm=0.0,
                   eta=cfg.solver.local_tol_fraction, local_max_iters=4096)
    assert np.array_equal(u_cycle, u_manual)
    np.testing.assert_allclose(u_cycle, G["kat_vcycle_u"], rtol=0, atol=1e-10)


def test_fine_unit_accounting():
    """tests/test_multigrid.py:298-302: fine_smoother_iterations == (nu_pre + nu_post) * iterations."""
    m, k = oracle.seeded_problem(128, 128, 0.05, 1)
    cfg = bp.MultigridConfig()
    _, rep = bp.fmg_solve(bp.build_hierarchy(bp.InpaintingProblem(m, k), cfg), cfg)
    assert rep.fine_smoother_iterations == (cfg.nu_pre + cfg.nu_post) * rep.iterations
    assert [rep.iterations, rep.fine_smoother_iterations] == list(G["kat_units"])
    for pre, post in ((2, 1), (0, 2), (3, 0)):
        c2 = bp.MultigridConfig(nu_pre=pre, nu_post=post)
        _, r2 = bp.fmg_solve(bp.build_hierarchy(bp.InpaintingProblem(m, k), c2), c2)
        assert r2.fine_smoother_iterations == (pre + post) * r2.iterations and r2.converged


def _robin_axis(n, left_diag, right_diag):
    t = 2.0 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    t[0, 0], t[-1, -1] = left_diag, right_diag
    return np.linalg.eigh(t)


@pytest.mark.parametrize("ratio", [1e-8, 1e-10, 1e-12, 1e-14])
@pytest.mark.parametrize("side", ["stop", "continue"])
def test_one_reduction_cg_identity_against_direct_rr(ratio, side):
    """The block-solve kernels evaluate the local CG stop test with
        |r - a q|^2 = |r|^2 - 2 a (r.q) + a^2 (q.q)
    (one reduction per step) where the reference forms r.r afresh (solvers.py:352-354).  The identity
    loses digits as rs_new / rs_k shrinks; this pins it where it is hardest: ONE CG step that reduces the
    squared residual by `ratio` (a residual made of two eigenvectors of the block's local operator), with
    the target 5 % above (`stop`) or below (`continue`) the true new value.  The decision and the
    correction must be those of the oracle's direct r.r (1e-14 is where 5 % stops being safe)."""
    n, img = 26, 58                      # block 0 of a 2 x 2 partition; only [0, 26)^2 is unknown
    mask = np.ones((img, img), dtype=bool)
    mask[:n, :n] = False
    # local operator on the free pixels: reflecting image border (diag 1), known neighbour on the other side (diag 2)
    lam, vec = _robin_axis(n, 1.0, 2.0)
    e1 = np.outer(vec[:, 0], vec[:, 0])                  # eigenvalue 2 * lam[0]
    e2 = np.outer(vec[:, 1], vec[:, 0])                  # eigenvalue lam[1] + lam[0]
    l1, l2 = 2.0 * lam[0], lam[0] + lam[1]
    eps = np.sqrt(ratio) / abs(1.0 - l2 / l1)            # rs_new / rs_k ~ eps^2 (1 - l2/l1)^2
    b = np.zeros((img, img))
    b[:n, :n] = 100.0 * (e1 + eps * e2)
    u = np.zeros((img, img))
    # one exact CG step in extended precision gives the true ratio the target is placed around
    r0 = (b[:n, :n]).astype(np.longdouble)
    q = (100.0 * (l1 * e1 + eps * l2 * e2)).astype(np.longdouble)
    a = (r0 * r0).sum() / (r0 * q).sum()
    r1 = r0 - a * q
    true_ratio = float((r1 * r1).sum() / (r0 * r0).sum())
    assert 0.3 * ratio < true_ratio < 3.0 * ratio
    eta = true_ratio * (1.05 if side == "stop" else 0.95)
    part = bp.build_partition(img, img, 32, 6)
    bs = bp.BlockSolver(mask, 1.0, part, bp.build_weights(part), alpha=0.5)
    op = bp.StencilOperator(mask, 1.0)
    got = u.copy()
    sweeps, rn = bp.oras_sweeps(op, bs, b, got, max_sweeps=1, stop_norm=0.0, eta=eta, local_max_iters=4096)
    want = u.copy()
    so, rno = oracle.oras_sweeps(mask, 1.0, 32, 6, 0.5, b, want, max_sweeps=1, stop_norm=0.0, eta=eta,
                                 local_max_iters=4096)
    assert sweeps == so == 1
    # a second CG step would change the correction by ~ 100 eps / l2: orders of magnitude above 1e-9
    second_step = 100.0 * eps / l2
    assert second_step > 1e-6
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-9 * max(1.0, np.abs(want).max()))
    if side == "stop":          # after the second step both residuals are rounding noise
        assert rn == pytest.approx(rno, rel=1e-6)
    else:
        assert max(rn, rno) < max(1e-4 * 100.0 * eps, 1e-6)
    # which of the two possible corrections is it: one CG step (a r0) or two (the exact local solution)?
    v1 = np.asarray(a * r0, dtype=np.float64)
    v2 = 100.0 * (e1 / l1 + eps * e2 / l2)
    stopped = np.abs(got[:n, :n] - v1).max() < np.abs(got[:n, :n] - v2).max()
    assert stopped == (side == "stop")
