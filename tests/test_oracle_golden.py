"""Pins the CPU oracle (oracle/fmg_oracle.c) against golden vectors written by
the reference itself (tests/golden/make_golden.py).  Runs anywhere (CPU)."""

import json
import os

import numpy as np
import pytest

import oracle

G = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(G, "golden_small.npz"))


@pytest.fixture(scope="module")
def meta():
    with open(os.path.join(G, "golden_small.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("i", range(4))
def test_stencil_and_transfers(gold, i):
    m, u, b, rhs, ce = (gold[f"t{i}_{k}"] for k in ("mask", "u", "b", "rhs", "ce"))
    # element-wise kernels keep the reference's operation order: bit-exact
    assert np.array_equal(oracle.apply_operator(m, 2.0, u), gold[f"t{i}_apply"])
    assert np.array_equal(oracle.residual(m, 1.0, b, u), gold[f"t{i}_residual"])
    cm = oracle.downsample_mask(m)
    assert np.array_equal(cm, gold[f"t{i}_cmask"])
    assert np.array_equal(oracle.downsample_values_modified(m, cm, rhs), gold[f"t{i}_val_mod"])
    assert np.array_equal(oracle.downsample_values_naive(m, rhs), gold[f"t{i}_val_naive"])
    assert np.array_equal(oracle.restrict_residual(u, cm), gold[f"t{i}_restrict"])
    assert np.array_equal(oracle.prolongate_correction(ce, m), gold[f"t{i}_pro_corr"])
    assert np.array_equal(oracle.prolongate_solution(ce, m, rhs), gold[f"t{i}_pro_sol"])


@pytest.mark.parametrize("j", range(10))
def test_partition_and_weights(gold, j):
    dim, bs, ov = (int(x) for x in gold[f"p{j}_cfg"])
    part = oracle.build_partition(dim, dim, bs, ov)
    assert np.array_equal(part.xs, gold[f"p{j}_xs"])
    wx, _ = oracle.build_weights(part)
    assert np.array_equal(wx, gold[f"p{j}_wx"])


@pytest.mark.parametrize("bs,ov", [(32, 6), (16, 2)])
def test_oras_sweeps_and_block_solves(gold, bs, ov):
    m, k = oracle.seeded_problem(80, 56, 0.15, 8)
    b = np.where(m, k[0], 0.0)
    u = b.copy()
    sweeps, rn = oracle.oras_sweeps(m, 1.0, bs, ov, 0.5, b, u, max_sweeps=3)
    hist = gold[f"sweep_{bs}_{ov}_hist"]
    assert sweeps == len(hist) - 1 == 3
    assert rn == pytest.approx(hist[-1], rel=1e-10)
    np.testing.assert_allclose(u, gold[f"sweep_{bs}_{ov}_u"], rtol=0, atol=1e-10)
    r = oracle.residual(m, 1.0, b, b)
    v = oracle.solve_blocks(m, 1.0, bs, ov, 0.5, r, 1e-5 * float(np.vdot(r, r)), 4 * min(bs, 80) * min(bs, 56))
    np.testing.assert_allclose(v, gold[f"blocks_{bs}_{ov}_v"], rtol=0, atol=1e-11)


@pytest.mark.parametrize("name", ["c64", "c80x56", "c97x131", "c20x30", "c256"])
def test_whole_path(gold, meta, name):
    c = meta[name]
    m, k = oracle.seeded_problem(c["w"], c["h"], c["density"], c["seed"], c["channels"])
    cfg = oracle.MultigridConfig(solver=oracle.SolverConfig(**c["solver"]), **c["mg"])
    hier = oracle.build_hierarchy(m, k, 1.0, cfg)
    assert len(hier) == int(gold[f"{name}_nlevels"])
    np.testing.assert_allclose(hier.levels[-1].rhs, gold[f"{name}_coarsest_rhs"], rtol=0, atol=1e-11)
    np.testing.assert_allclose(oracle.cascadic_init(hier, cfg, 0), gold[f"{name}_cascade"], rtol=0, atol=1e-7)
    out, reps = oracle.solve_image(m, k, 1.0, cfg)
    for r, g in zip(reps, c["reports"]):
        assert r.iterations == g["iterations"]
        assert r.fine_smoother_iterations == g["fine_units"]
        assert r.converged == g["converged"]
        assert r.baseline_residual == pytest.approx(g["baseline"], rel=1e-12)
        # residuals far below the stopping tolerance are summation-order noise: compare on its scale
        floor = 1e-6 * cfg.solver.tol_rel
        assert r.final_rel_residual == pytest.approx(g["final_rel"], rel=1e-6, abs=floor)
        np.testing.assert_allclose(r.history, g["history"], rtol=1e-6, atol=floor)
    # north_star bar is 1e-3; the oracle sits many orders below it
    assert np.abs(out - gold[f"{name}_fields"]).max() <= 1e-7


def test_anchors_if_present():
    """1080p / 4K anchors (V-cycles, final residual, a strided sample of the reference field)."""
    p = os.path.join(G, "anchors.json")
    if not os.path.exists(p):
        pytest.skip("anchors not generated")
    with open(p) as f:
        anchors = json.load(f)
    sample = np.load(os.path.join(G, "anchors_sample.npz"))
    a = anchors["1080p_4pct_16_2"]
    m, k = oracle.seeded_problem(a["w"], a["h"], a["density"], 0, a["channels"])
    out, reps = oracle.solve_image(m, k, 1.0, oracle.MultigridConfig(block_size=16, overlap=2))
    for r, g in zip(reps, a["reports"]):
        assert r.iterations == g["iterations"]
        assert r.final_rel_residual == pytest.approx(g["final_rel"], rel=1e-6)
    got = out.reshape(a["channels"], -1)[:, ::997]
    assert np.abs(got - sample["1080p_4pct_16_2"]).max() <= 1e-6


# ---- the five comparison pipelines (golden_pipelines.*: written by the reference) -------------

@pytest.fixture(scope="module")
def pgold():
    return np.load(os.path.join(G, "golden_pipelines.npz"))


@pytest.fixture(scope="module")
def pmeta():
    with open(os.path.join(G, "golden_pipelines.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("solver", ["ml-oras", "oras", "mg-cg", "ml-cg", "cg"])
@pytest.mark.parametrize("case", ["q96x64", "q160x120", "q20x30", "q128cap"])
def test_comparison_pipelines(pgold, pmeta, case, solver):
    """oracle ml-oras / oras / mg-cg / ml-cg / cg == the reference's own outputs (pipelines.py:20-114)."""
    c = pmeta[case]
    m, k = oracle.seeded_problem(c["w"], c["h"], c["density"], c["seed"], channels=c["channels"])
    scfg = oracle.SolverConfig(**c["solver"])
    bs, ov = c["mg"]["block_size"], c["mg"]["overlap"]
    base = solver.split("-")[-1]
    got = []
    if "-" in solver:
        mode = "multilevel" if solver.startswith("ml") else "full_multigrid"
        fields, reps = oracle.solve_image(m, k, 1.0, oracle.MultigridConfig(
            block_size=bs, overlap=ov, smoother=base, mode=mode, solver=scfg))
        got = [(fields[ch], dict(iterations=r.iterations, final_rel=r.final_rel_residual,
                                 fine_units=r.fine_smoother_iterations, converged=r.converged,
                                 history=r.history, baseline=r.baseline_residual))
               for ch, r in enumerate(reps)]
    else:
        for ch in range(c["channels"]):
            if base == "cg":
                u, r = oracle.cg_solve(m, k[ch], 1.0, scfg)
                rep = dict(iterations=r.iterations, final_rel=r.final_rel_residual,
                           fine_units=r.fine_smoother_iterations, converged=r.converged,
                           history=r.history, baseline=r.baseline_residual)
            else:
                u, r = oracle.oras_solve(m, k[ch], 1.0, bs, ov, scfg)
                rep = dict(iterations=r["iterations"], final_rel=r["final_rel_residual"],
                           fine_units=r["fine_smoother_iterations"], converged=r["converged"],
                           history=r["history"], baseline=r["baseline_residual"])
            got.append((u, rep))
    for ch, (u, rep) in enumerate(got):
        want = c["reports"][solver][ch]
        assert (rep["iterations"], rep["fine_units"], bool(rep["converged"])) == \
               (want["iterations"], want["fine_units"], want["converged"])
        assert rep["final_rel"] == pytest.approx(want["final_rel"], rel=1e-6, abs=1e-13)
        assert rep["baseline"] == pytest.approx(want["baseline"], rel=1e-12)
        np.testing.assert_allclose(rep["history"], want["history"], rtol=1e-6, atol=1e-13)
        np.testing.assert_allclose(u, pgold[f"{case}_{solver}_fields"][ch], rtol=0, atol=1e-9)


def test_eight_bit_decode_vectors_are_reproduced_by_the_oracle():
    """golden_images.* (fileio.image_from_fields of the reference's mg-oras solve): the oracle's fields
    quantise to the reference's bytes, and the stored P4 raster is np.packbits of the stored mask."""
    g = np.load(os.path.join(G, "golden_images.npz"))
    with open(os.path.join(G, "golden_images.json")) as f:
        cases = json.load(f)
    assert np.array_equal(np.packbits(g["raster_mask"], axis=1), g["raster_bytes"])
    assert np.array_equal(np.unpackbits(g["raster_bytes"], axis=1)[:, : g["raster_mask"].shape[1]].astype(bool),
                          g["raster_mask"])
    for name in ("quant_rgb", "quant_gray"):
        q = np.clip(np.round(g[f"{name}_fields"]), 0, 255).astype(np.uint8)
        want = g[f"{name}_pixels"]
        assert np.array_equal(q[0] if q.shape[0] == 1 else np.moveaxis(q, 0, 2), want)
    for name, c in cases.items():
        m, k = oracle.seeded_problem(c["w"], c["h"], c["density"], c["seed"], channels=c["channels"])
        assert np.array_equal(k, k.astype(np.uint8).astype(np.float64))      # the inputs are 8-bit images
        cfg = oracle.MultigridConfig(block_size=c["block_size"], overlap=c["overlap"],
                                     solver=oracle.SolverConfig(**c.get("solver", {})))
        fields, reps = oracle.solve_image(m, k, 1.0, cfg)
        assert [r.iterations for r in reps] == c["iterations"]
        q = np.clip(np.round(fields), 0, 255).astype(np.uint8)
        assert np.array_equal(q[0] if c["channels"] == 1 else np.moveaxis(q, 0, 2), g[f"{name}_pixels"])
