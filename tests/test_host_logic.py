"""CPU tests: the C-ABI library loads and exports every declared symbol, the
host-side geometry matches the reference's known answers and the oracle, and
the Python mirror validates like the reference.  No compute calls (no GPU)."""

import ctypes as C
import os
import re

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import oracle
import paper_2401_06744_b200 as bp
from paper_2401_06744_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "b200paint.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    declared = set(re.findall(r"\b(b200p_[a-z0-9_]+)\s*\(", hdr))
    assert len(declared) >= 40
    lib = C.CDLL(_lib.LIB_PATH)
    missing = [n for n in sorted(declared) if not hasattr(lib, n)]
    assert not missing, missing
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(_lib.B200PaintError):
        bp.Plan(64, 64)
    m = np.zeros((32, 32), bool)
    m[1, 1] = True
    with pytest.raises(_lib.B200PaintError):
        bp.solve_image(bp.InpaintingProblem(m, np.zeros((32, 32))), "mg-oras")
    # the C-ABI itself: valid config, no device -> a CUDA error code (> 0), never a result
    cfg = _lib.Config()
    _lib.lib().b200p_config_default(C.byref(cfg), 64, 64, 1)
    h = C.c_void_p()
    rc = _lib.lib().b200p_plan_create(C.byref(cfg), C.byref(h))
    assert rc > 0 and not h.value
    assert _lib.last_error()


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2401_06744_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", text, flags=re.M), f
                assert "liboracle" not in text and "fmg_oracle" not in text, f


@pytest.mark.parametrize("bad", [
    dict(width=0), dict(height=-1), dict(channels=0), dict(frames=0), dict(spacing=0.0),
    dict(block_size=6, overlap=6), dict(overlap=-1), dict(block_size=128, overlap=6),
    dict(nu_pre=0, nu_post=0), dict(tol_rel=0.0), dict(tol_rel=1.0), dict(alpha=0.0), dict(eta=0.0),
    dict(value_downsampling=2),
])
def test_plan_create_rejects_bad_configs_before_touching_cuda(bad):
    cfg = _lib.Config()
    _lib.lib().b200p_config_default(C.byref(cfg), 64, 48, 3)
    for k, v in bad.items():
        setattr(cfg, k, v)
    h = C.c_void_p()
    rc = _lib.lib().b200p_plan_create(C.byref(cfg), C.byref(h))
    assert rc in (_lib.ERR_ARG, _lib.ERR_UNSUPPORTED) and not h.value


def test_config_defaults_match_reference_defaults():
    cfg = _lib.Config()
    _lib.lib().b200p_config_default(C.byref(cfg), 3840, 2160, 3)
    m, s = bp.MultigridConfig(), bp.SolverConfig()
    assert (cfg.block_size, cfg.overlap, cfg.nu_pre, cfg.nu_post, cfg.v_cycles_max) == \
        (m.block_size, m.overlap, m.nu_pre, m.nu_post, m.v_cycles_max)
    assert (cfg.coarse_tol, cfg.coarse_max_iters, cfg.tol_rel, cfg.alpha, cfg.eta) == \
        (m.coarse_tol, m.coarse_max_iters, s.tol_rel, s.alpha, s.local_tol_fraction)
    assert cfg.value_downsampling == 1 and cfg.local_max_iters == 0


# ---- geometry known answers (tests/test_partition.py, tests/test_multigrid.py of the reference) ----

def test_4k_partition_and_levels():
    p = bp.build_partition(3840, 2160, 32, 6)
    assert (p.nx, p.ny, p.nblocks) == (148, 83, 12284)              # tests/test_partition.py:26-30
    assert list(bp.build_partition(64, 64, 32, 6).xs) == [0, 26, 32]  # :39-43
    info = (_lib.LevelInfo * 32)()
    n = _lib.lib().b200p_level_shapes(3840, 2160, 1.0, 32, 6, info, 32)
    assert n == 8 and (info[7].height, info[7].width) == (17, 30)  # tests/test_multigrid.py:182-188
    assert [info[i].spacing for i in range(n)] == [2.0 ** i for i in range(n)]
    n = _lib.lib().b200p_level_shapes(256, 256, 1.0, 32, 6, info, 32)
    assert n == 4                                                   # tests/test_multigrid.py:194-199
    n = _lib.lib().b200p_level_shapes(20, 30, 1.0, 32, 6, info, 32)
    assert n == 1 and (info[0].block_w, info[0].block_h, info[0].nx, info[0].ny) == (20, 30, 1, 1)


def test_ramp_values_and_clamped_renormalisation():
    p = bp.build_partition(200, 200, 32, 6)
    w = bp.build_weights(p)
    np.testing.assert_allclose(w.wx[1][:6], [0, .2, .4, .6, .8, 1.0], atol=1e-15)  # tests/test_partition.py:76-82
    np.testing.assert_allclose(w.wx[1][-6:], [1.0, .8, .6, .4, .2, 0], atol=1e-15)
    assert w.wx[0][0] == 1.0 and w.wx[-1][-1] == 1.0                # image-border sides stay at 1
    p2 = bp.build_partition(64, 64, 16, 2)                          # SURVEY: binary ramp, 0.5/0.5 at the clamp
    w2 = bp.build_weights(p2)
    assert set(np.unique(w2.wx[:-2])) <= {0.0, 1.0}
    rect = p.rect(p.nx + 1)
    assert (rect.x0, rect.y0, rect.inner_left, rect.inner_top) == (26, 26, True, True)
    with pytest.raises(ValueError):
        bp.build_partition(0, 10)
    with pytest.raises(ValueError):
        bp.build_partition(10, 10, 8, 8)


@settings(max_examples=150, deadline=None)
@given(dim=st.integers(1, 400), block=st.integers(2, 64), data=st.data())
def test_partition_covers_and_weights_sum_to_one(dim, block, data):
    overlap = data.draw(st.integers(0, block - 1))
    if overlap == 1:
        overlap = 0  # overlap 1 yields NaN weights in the reference as well
    p = bp.build_partition(dim, dim, block, overlap)
    o = oracle.build_partition(dim, dim, block, overlap)
    assert np.array_equal(p.xs, o.xs)
    assert p.xs[0] == 0 and p.xs[-1] + p.block_w == dim and (np.diff(p.xs) > 0).all()
    assert (np.diff(p.xs) <= p.block_w).all()                       # no gaps
    w = bp.build_weights(p)
    assert np.array_equal(w.wx, oracle.build_weights(o)[0])
    total = np.zeros(dim)
    for i, s in enumerate(p.xs):
        total[s:s + p.block_w] += w.wx[i]
    np.testing.assert_allclose(total, 1.0, atol=1e-12)              # tests/test_partition.py:99-121


# ---- the Python mirror validates like the reference ----

def test_config_validation():
    for kw in (dict(nu_pre=0, nu_post=0), dict(smoother="jacobi"), dict(mode="w-cycle"),
               dict(value_downsampling="median")):
        with pytest.raises(ValueError):
            bp.MultigridConfig(**kw)
    for kw in (dict(tol_rel=0.0), dict(tol_rel=1.5), dict(alpha=0.0), dict(local_tol_fraction=0.0)):
        with pytest.raises(ValueError):
            bp.SolverConfig(**kw)
    assert bp.split_solver_name("mg-oras") == ("oras", "full_multigrid")
    assert bp.split_solver_name("cg") == ("cg", "single")
    assert bp.join_solver_name("oras", "multilevel") == "ml-oras"
    with pytest.raises(ValueError):
        bp.split_solver_name("fmg")


def test_problem_validation():
    m = np.zeros((4, 5), bool)
    with pytest.raises(ValueError):
        bp.InpaintingProblem(m, np.zeros((4, 4)))
    with pytest.raises(ValueError):
        bp.InpaintingProblem(m, np.zeros((2, 3, 4, 5)))
    with pytest.raises(ValueError):
        bp.InpaintingProblem(m, np.full((4, 5), np.inf))
    with pytest.raises(ValueError):
        bp.InpaintingProblem(m, np.zeros((4, 5)), spacing=0.0)
    p = bp.InpaintingProblem(m, np.ones((4, 5)))
    assert p.channels == 1 and p.shape == (4, 5) and p.known.shape == (1, 4, 5)
    assert not p.rhs(0).any()
    assert bp.compute_metrics(np.zeros(4), np.zeros(4)).psnr == np.inf
    assert bp.compute_metrics(np.zeros(4), np.full(4, 255.0)).psnr == pytest.approx(0.0)


def test_synthetic_inputs_match_oracle_recipe():
    from paper_2401_06744_b200 import synthetic
    for w, h, d, s in [(64, 48, 0.1, 0), (256, 256, 0.05, 3)]:
        m, k = synthetic.seeded_problem(w, h, d, s, 2)
        mo, ko = oracle.seeded_problem(w, h, d, s, 2)
        assert np.array_equal(m, mo) and np.array_equal(k, ko)
        assert int(m.sum()) == int(round(d * w * h))
    ms, ks = synthetic.seeded_frames(32, 24, 0.2, 3, 2, first_seed=5)
    assert ms.shape == (3, 24, 32) and ks.shape == (3, 2, 24, 32)
    assert np.array_equal(ms[1], synthetic.random_mask(32, 24, 0.2, 6))


def test_report_csv_matches_the_reference_writer(tmp_path, diffpaint):
    """suites.format_report_csv == fileio.write_report_csv (fileio.py:233-275) byte for byte."""
    from paper_2401_06744_b200 import suites
    rows = [
        {"solver": "mg-oras", "width": 3840, "height": 2160, "density": 0.02, "seed": 0, "alpha": 0.5, "tol": 1e-3,
         "iterations": 2, "rel_residual": 1.2895951277968e-4, "mse_vs_reference": 3.25e-7, "psnr": 112.98765,
         "wall_time_s": 0.0035801},
        {"solver": "ml-oras+naive", "width": 256, "height": 256, "density": 0.0123456789, "seed": 3, "alpha": 2.0,
         "tol": 1e-10, "iterations": 17, "rel_residual": 9.9e-11, "mse_vs_reference": None, "psnr": None,
         "wall_time_s": 1.5},
        {"solver": "cg", "width": 20, "height": 30, "density": 0.2, "seed": 1, "alpha": 0.5, "tol": 1e-6,
         "iterations": 100, "rel_residual": 0.5, "mse_vs_reference": 0.0, "psnr": float("inf"), "wall_time_s": 2},
    ]
    from diffpaint import fileio
    path = tmp_path / "ref.csv"
    fileio.write_report_csv(path, rows)
    assert suites.format_report_csv(rows) == open(path, newline="").read()
    assert suites.CSV_HEADER == fileio.CSV_HEADER and suites.ROW_FIELDS == fileio.CSV_FIELDS
    mine = tmp_path / "mine.csv"
    suites.write_report_csv(mine, rows)
    assert open(mine, "rb").read() == open(path, "rb").read()


def test_direct_truth_matches_the_reference_dense_oracle(diffpaint):
    """suites.direct_truth (sparse LU) == oracle.solve (dense LU, oracle.py:38-80) on small problems."""
    from paper_2401_06744_b200 import suites
    for (w, h, dens, seed, ch, spacing) in [(24, 17, 0.15, 1, 1, 1.0), (31, 40, 0.05, 2, 3, 0.5), (8, 8, 0.5, 3, 1, 2.0)]:
        m, k = oracle.seeded_problem(w, h, dens, seed, channels=ch)
        got = suites.direct_truth(bp.InpaintingProblem(m, k, spacing))
        ref_prob = diffpaint.InpaintingProblem(m, k, spacing)
        from diffpaint import oracle as dense
        want = np.stack([dense.solve(ref_prob, c) for c in range(ch)])
        assert np.abs(got - want).max() <= 1e-9
    with pytest.raises(bp.EmptyMaskError):
        suites.direct_truth(bp.InpaintingProblem(np.zeros((4, 4), bool), np.zeros((1, 4, 4))))
    with pytest.raises(ValueError, match="refusing"):
        suites.direct_truth(bp.InpaintingProblem(np.ones((200, 200), bool), np.zeros((1, 200, 200))))


def test_block_restriction_and_weighted_extension_like_the_reference(diffpaint):
    """partition.py:171-188: restrict_to_block copies, extend_add_weighted(field, rect, weights, local)
    accumulates in place, both refuse blocks outside the field; sum_i R_i^T (w_i * R_i u) == u."""
    from diffpaint import partition as rp
    part, rpart = bp.build_partition(70, 45, 16, 4), rp.build_partition(70, 45, 16, 4)
    wts, rw = bp.build_weights(part), rp.build_weights(rpart)
    u = np.random.default_rng(3).normal(size=(45, 70))
    acc, racc = np.zeros_like(u), np.zeros_like(u)
    for i, (rect, rrect) in enumerate(zip(part.rects(), rpart.rects())):
        loc, rloc = bp.restrict_to_block(u, rect), rp.restrict_to_block(u, rrect)
        assert np.array_equal(loc, rloc) and loc.base is None          # a copy, not a view
        bp.extend_add_weighted(field=acc, rect=rect, weights=wts.block(part, i), local=loc)
        rp.extend_add_weighted(racc, rrect, rw.block(rpart, i), rloc)
    assert np.array_equal(acc, racc) and np.abs(acc - u).max() <= 1e-12
    bad = bp.BlockRect(60, 40, 16, 16, True, False, True, False)
    with pytest.raises(ValueError, match="exceeds field bounds"):
        bp.restrict_to_block(u, bad)
    with pytest.raises(ValueError, match="exceeds field bounds"):
        bp.extend_add_weighted(acc, bad, np.ones((16, 16)), np.ones((16, 16)))
    with pytest.raises(ValueError, match="do not match the block extent"):
        bp.extend_add_weighted(acc, part.rect(0), np.ones((3, 3)), np.ones((16, 16)))
