"""The CUDA path against the golden vectors WRITTEN BY THE REFERENCE (tests/golden/, generator
make_golden.py) -- no oracle in between.  Runs on the GPU box, where /root/reference does not exist."""

import json
import os

import numpy as np
import pytest

import paper_2401_06744_b200 as bp
from paper_2401_06744_b200 import synthetic

pytestmark = pytest.mark.gpu

G = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(G, "golden_small.npz"))


@pytest.fixture(scope="module")
def meta():
    with open(os.path.join(G, "golden_small.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("i", range(4))
def test_stencil_and_transfers_vs_reference_vectors(gold, i):
    m, u, b, rhs, ce = (gold[f"t{i}_{k}"] for k in ("mask", "u", "b", "rhs", "ce"))
    np.testing.assert_allclose(bp.StencilOperator(m, 2.0).apply(u), gold[f"t{i}_apply"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(bp.StencilOperator(m, 1.0).residual(b, u), gold[f"t{i}_residual"], rtol=0, atol=1e-10)
    cm = bp.downsample_mask(m)
    assert np.array_equal(cm, gold[f"t{i}_cmask"])                      # byte work: bit-exact
    np.testing.assert_allclose(bp.downsample_values_modified(m, cm, rhs), gold[f"t{i}_val_mod"], rtol=0, atol=1e-11)
    np.testing.assert_allclose(bp.downsample_values_naive(m, rhs), gold[f"t{i}_val_naive"], rtol=0, atol=1e-11)
    np.testing.assert_allclose(bp.restrict_residual(u, cm), gold[f"t{i}_restrict"], rtol=0, atol=1e-11)
    np.testing.assert_allclose(bp.prolongate_correction(ce, m), gold[f"t{i}_pro_corr"], rtol=0, atol=1e-11)
    np.testing.assert_allclose(bp.prolongate_solution(ce, m, rhs), gold[f"t{i}_pro_sol"], rtol=0, atol=1e-11)


@pytest.mark.parametrize("j", range(10))
def test_partition_and_weights_vs_reference_vectors(gold, j):
    dim, bs, ov = (int(x) for x in gold[f"p{j}_cfg"])
    part = bp.build_partition(dim, dim, bs, ov)
    assert np.array_equal(np.asarray(part.xs), gold[f"p{j}_xs"])        # index work: bit-exact
    wx = bp.build_weights(part).wx
    assert np.array_equal(np.asarray(wx), gold[f"p{j}_wx"])


@pytest.mark.parametrize("bs,ov", [(32, 6), (16, 2)])
def test_oras_sweeps_vs_reference_vectors(gold, bs, ov):
    m, k = synthetic.seeded_problem(80, 56, 0.15, 8)
    b = np.where(m, k[0], 0.0)
    u = b.copy()
    part = bp.build_partition(80, 56, bs, ov)
    blocks = bp.BlockSolver(m, 1.0, part, bp.build_weights(part), 0.5)
    hist = []
    sweeps, rn = bp.oras_sweeps(bp.StencilOperator(m, 1.0), blocks, b, u, max_sweeps=3, stop_norm=0.0, eta=1e-5,
                                local_max_iters=None, on_state=lambda uu, r, it: hist.append(r))
    want = gold[f"sweep_{bs}_{ov}_hist"]
    assert sweeps == len(want) - 1 == 3
    np.testing.assert_allclose(hist, want, rtol=1e-9)
    np.testing.assert_allclose(u, gold[f"sweep_{bs}_{ov}_u"], rtol=0, atol=1e-8)


@pytest.mark.parametrize("name", ["c64", "c80x56", "c97x131", "c20x30", "c256"])
def test_whole_path_vs_reference_vectors(gold, meta, name):
    c = meta[name]
    m, k = synthetic.seeded_problem(c["w"], c["h"], c["density"], c["seed"], c["channels"])
    cfg = bp.MultigridConfig(solver=bp.SolverConfig(**c["solver"]), **c["mg"])
    prob = bp.InpaintingProblem(m, k)
    hier = bp.build_hierarchy(prob, cfg)
    assert len(hier) == int(gold[f"{name}_nlevels"])
    np.testing.assert_allclose(bp.cascadic_init(hier, cfg, 0), gold[f"{name}_cascade"], rtol=0, atol=1e-7)
    res = bp.solve_image(prob, "mg-oras", cfg)
    for r, g in zip(res.reports, c["reports"]):
        assert r.iterations == g["iterations"]
        assert r.fine_smoother_iterations == g["fine_units"]
        assert r.converged == g["converged"]
        assert r.baseline_residual == pytest.approx(g["baseline"], rel=1e-12)
        floor = 1e-6 * cfg.solver.tol_rel
        assert r.final_rel_residual == pytest.approx(g["final_rel"], rel=1e-6, abs=floor)
        np.testing.assert_allclose(r.history, g["history"], rtol=1e-6, atol=floor)
    # the north star's bar is 1e-3 on [0, 255]; the CUDA path sits many orders below it
    assert np.abs(res.fields - gold[f"{name}_fields"]).max() <= 1e-7


@pytest.mark.parametrize("name,bs,ov", [("1080p_4pct_16_2", 16, 2), ("4k_2pct_32_6", 32, 6), ("4k_0.5pct_32_6", 32, 6)])
def test_full_size_anchors_vs_reference_vectors(name, bs, ov):
    """BASELINE configs[1..3] at FULL size: V-cycles, final residuals and a strided sample of the field the
    REFERENCE produced (tests/golden/anchors*.{json,npz}); max-abs bar 1e-3, measured ~1e-9."""
    with open(os.path.join(G, "anchors.json")) as f:
        a = json.load(f)[name]
    sample = np.load(os.path.join(G, "anchors_sample.npz"))
    m, k = synthetic.seeded_problem(a["w"], a["h"], a["density"], 0, a["channels"])
    res = bp.solve_image(bp.InpaintingProblem(m, k), "mg-oras", bp.MultigridConfig(block_size=bs, overlap=ov))
    for r, g in zip(res.reports, a["reports"]):
        assert r.iterations == g["iterations"]
        assert r.final_rel_residual == pytest.approx(g["final_rel"], rel=1e-6)
    got = res.fields.reshape(a["channels"], -1)[:, ::997]
    assert got.shape == sample[name].shape
    assert np.abs(got - sample[name]).max() <= 1e-6


@pytest.mark.parametrize("solver", ["ml-oras", "oras", "mg-cg", "ml-cg", "cg"])
@pytest.mark.parametrize("case", ["q96x64", "q160x120", "q20x30", "q128cap"])
def test_comparison_pipelines_vs_reference_vectors(case, solver):
    with open(os.path.join(G, "golden_pipelines.json")) as f:
        c = json.load(f)[case]
    pg = np.load(os.path.join(G, "golden_pipelines.npz"))
    m, k = synthetic.seeded_problem(c["w"], c["h"], c["density"], c["seed"], channels=c["channels"])
    cfg = bp.MultigridConfig(block_size=c["mg"]["block_size"], overlap=c["mg"]["overlap"],
                             solver=bp.SolverConfig(**c["solver"]))
    res = bp.solve_image(bp.InpaintingProblem(m, k), solver, cfg)
    for ch, r in enumerate(res.reports):
        want = c["reports"][solver][ch]
        assert (r.iterations, r.fine_smoother_iterations, bool(r.converged)) == \
               (want["iterations"], want["fine_units"], want["converged"])
        assert r.final_rel_residual == pytest.approx(want["final_rel"], rel=1e-6, abs=1e-13)
        assert r.baseline_residual == pytest.approx(want["baseline"], rel=1e-12)
        np.testing.assert_allclose(r.history, want["history"], rtol=1e-6, atol=1e-13)
    np.testing.assert_allclose(res.fields, pg[f"{case}_{solver}_fields"], rtol=0, atol=1e-8)
