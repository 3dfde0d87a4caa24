"""Generates the golden fixtures in this directory from the LIVE reference
(`/root/reference/pkg/src/diffpaint`, pure Python/NumPy).  Run in the build
container (the reference is not present on the GPU box):

    python tests/golden/make_golden.py            # small vectors  (seconds)
    python tests/golden/make_golden.py --anchors  # + 1080p / 4K anchors (~3 min)
    python tests/golden/make_golden.py --pipelines  # only golden_pipelines.* (comparison pipelines)
    python tests/golden/make_golden.py --images     # only golden_images.* (8-bit decode, P4 raster, quantiser)

Outputs: golden_small.npz (inputs are regenerated from seeds by the tests; only
reference OUTPUTS are stored) and anchors.json / anchors_4k_sample.npz."""

import argparse
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
import diffpaint as dp  # noqa: E402
from diffpaint import multigrid as mg  # noqa: E402
from diffpaint import solvers as sv  # noqa: E402


def seeded(w, h, density, seed, channels=1):
    mask = dp.random_mask(w, h, density, seed)
    known = np.stack([dp.synthetic_image(w, h, seed + 1000 + c) for c in range(channels)])
    return dp.InpaintingProblem(mask, known)


def small():
    out = {}
    rng = np.random.default_rng(2401_06744)
    # inputs drawn here are stored too (they are not reproducible from a public seed recipe)
    for i, shape in enumerate([(8, 8), (7, 9), (8, 5), (33, 47)]):
        m = rng.random(shape) < 0.25
        m.flat[0] = True
        u = rng.normal(size=shape) * 100
        b = rng.normal(size=shape) * 100
        cs = ((shape[0] + 1) // 2, (shape[1] + 1) // 2)
        cm = mg.downsample_mask(m)
        rhs = np.where(m, np.round(rng.uniform(0, 255, size=shape)), 0.0)
        ce = rng.normal(size=cs)
        out[f"t{i}_mask"] = m
        out[f"t{i}_u"] = u
        out[f"t{i}_b"] = b
        out[f"t{i}_rhs"] = rhs
        out[f"t{i}_ce"] = ce
        out[f"t{i}_apply"] = dp.StencilOperator(m, 2.0).apply(u)
        out[f"t{i}_residual"] = dp.StencilOperator(m, 1.0).residual(b, u)
        out[f"t{i}_cmask"] = cm
        out[f"t{i}_val_mod"] = mg.downsample_values_modified(m, cm, rhs)
        out[f"t{i}_val_naive"] = mg.downsample_values_naive(m, rhs)
        out[f"t{i}_restrict"] = mg.restrict_residual(u, cm)
        out[f"t{i}_pro_corr"] = mg.prolongate_correction(ce, m)
        out[f"t{i}_pro_sol"] = mg.prolongate_solution(ce, m, rhs)
    # partitions / weights
    for j, (dim, bs, ov) in enumerate([(3840, 32, 6), (2160, 32, 6), (64, 32, 6), (80, 16, 2), (56, 32, 6),
                                       (20, 32, 6), (135, 32, 6), (100, 24, 4), (33, 32, 0), (1080, 16, 2)]):
        part = dp.build_partition(dim, dim, bs, ov)
        out[f"p{j}_cfg"] = np.array([dim, bs, ov])
        out[f"p{j}_xs"] = part.xs
        out[f"p{j}_wx"] = dp.build_weights(part).wx
    # ORAS sweeps and block solves on the clamped-block case of tests/test_solvers.py:156-169
    prob = seeded(80, 56, 0.15, 8)
    for bs, ov in [(32, 6), (16, 2)]:
        part = dp.build_partition(80, 56, bs, ov)
        blocks = sv.BlockSolver(prob.mask, 1.0, part, dp.build_weights(part), 0.5)
        b = prob.rhs(0)
        u = b.copy()
        hist = []
        sweeps, rn = sv.oras_sweeps(prob.operator(), blocks, b, u, max_sweeps=3, stop_norm=0.0, eta=1e-5,
                                    local_max_iters=4 * part.block_w * part.block_h,
                                    on_state=lambda uu, r, s: hist.append(r))
        out[f"sweep_{bs}_{ov}_u"] = u
        out[f"sweep_{bs}_{ov}_hist"] = np.array(hist)
        r = prob.operator().residual(b, b)
        out[f"blocks_{bs}_{ov}_v"] = blocks.solve_blocks(blocks.gather(r), 1e-5 * float(np.vdot(r, r)),
                                                        4 * part.block_w * part.block_h)
    # whole-path solves
    cases = {
        "c64": (64, 64, 0.10, 1, 1, dict(block_size=16, overlap=2), dict(tol_rel=1e-8)),
        "c80x56": (80, 56, 0.15, 8, 1, dict(block_size=32, overlap=6), dict(tol_rel=1e-6)),
        "c97x131": (97, 131, 0.03, 2, 2, dict(block_size=16, overlap=2), dict()),
        "c20x30": (20, 30, 0.20, 3, 1, dict(block_size=32, overlap=6), dict(tol_rel=1e-6)),
        "c256": (256, 256, 0.05, 0, 1, dict(block_size=16, overlap=2), dict()),
    }
    meta = {}
    for name, (w, h, dens, seed, ch, mkw, skw) in cases.items():
        prob = seeded(w, h, dens, seed, ch)
        cfg = dp.MultigridConfig(solver=dp.SolverConfig(**skw), **mkw)
        res = dp.solve_image(prob, "mg-oras", cfg)
        out[f"{name}_fields"] = res.fields
        meta[name] = dict(w=w, h=h, density=dens, seed=seed, channels=ch, mg=mkw, solver=skw,
                          reports=[dict(iterations=r.iterations, final_rel=r.final_rel_residual,
                                        baseline=r.baseline_residual, fine_units=r.fine_smoother_iterations,
                                        converged=bool(r.converged), history=list(r.history))
                                   for r in res.reports])
        hier = dp.build_hierarchy(prob, cfg)
        out[f"{name}_cascade"] = dp.cascadic_init(hier, cfg, 0)
        out[f"{name}_nlevels"] = np.array(len(hier))
        out[f"{name}_coarsest_rhs"] = hier.levels[-1].rhs
    np.savez_compressed(os.path.join(HERE, "golden_small.npz"), **out)
    with open(os.path.join(HERE, "golden_small.json"), "w") as f:
        json.dump(meta, f, indent=1)


def pipelines():
    """The five comparison pipelines (pipelines.py:20-39): ml-oras, oras, mg-cg, ml-cg, cg."""
    out, meta = {}, {}
    cases = {
        "q96x64": (96, 64, 0.10, 1, 2, dict(block_size=16, overlap=2), dict()),
        "q160x120": (160, 120, 0.05, 3, 1, dict(block_size=32, overlap=6), dict(tol_rel=1e-5)),
        "q20x30": (20, 30, 0.20, 3, 1, dict(block_size=32, overlap=6), dict(tol_rel=1e-6)),
        "q128cap": (128, 128, 0.05, 6, 1, dict(block_size=16, overlap=2), dict(max_outer_iters=4)),
    }
    for name, (w, h, dens, seed, ch, mkw, skw) in cases.items():
        prob = seeded(w, h, dens, seed, ch)
        cfg = dp.MultigridConfig(solver=dp.SolverConfig(**skw), **mkw)
        meta[name] = dict(w=w, h=h, density=dens, seed=seed, channels=ch, mg=mkw, solver=skw, reports={})
        for solver in ("ml-oras", "oras", "mg-cg", "ml-cg", "cg"):
            res = dp.solve_image(prob, solver, cfg)
            out[f"{name}_{solver}_fields"] = res.fields
            meta[name]["reports"][solver] = [
                dict(iterations=r.iterations, final_rel=r.final_rel_residual, baseline=r.baseline_residual,
                     fine_units=r.fine_smoother_iterations, converged=bool(r.converged), history=list(r.history))
                for r in res.reports]
    np.savez_compressed(os.path.join(HERE, "golden_pipelines.npz"), **out)
    with open(os.path.join(HERE, "golden_pipelines.json"), "w") as f:
        json.dump(meta, f, indent=1)


IMAGE_CASES = {
    # name: (w, h, density, seed, channels, block, overlap)
    "img_rgb_256x192": (256, 192, 0.03, 5, 3, 32, 6),      # warp-per-block sweep, fused 8-bit egress
    "img_gray_203x131": (203, 131, 0.05, 4, 1, 16, 2),     # odd width (raster rows padded), 16x16 blocks
    "img_gray_20x30": (20, 30, 0.20, 3, 1, 32, 6),         # single level: the tail pass writes the image
    "img_rgb_dense_64x48": (64, 48, 0.97, 9, 3, 16, 2),    # nearly everything known
    "img_rgb_loose_96x64": (96, 64, 0.10, 2, 3, 16, 2, dict(tol_rel=0.5)),  # multilevel, no V-cycle needed: tail pass
}


def images():
    """8-bit file path: ImageFile.channel_fields -> solve_image -> image_from_fields
    (fileio.py:51-65) and the P4 raster of write_mask (fileio.py:219-230), all by the reference."""
    import tempfile
    from diffpaint import fileio
    out, meta = {}, {}
    # quantiser known answers: ties (round half to even), out-of-range, exact integers
    rng = np.random.default_rng(65)
    special = np.array([0.5, 1.5, 2.5, 3.5, 126.5, 127.5, 253.5, 254.5, 255.5, -0.5, -0.4999, 255.4999, 1e6, -1e6,
                        0.0, 255.0, 17.0, 0.49999999999, 254.50000000001, -0.0])
    f3 = rng.uniform(-40.0, 300.0, size=(3, 16, 24))
    f3.reshape(-1)[: special.size * 3 : 3] = special
    f1 = np.floor(rng.uniform(-3.0, 259.0, size=(1, 9, 11))) + 0.5      # nothing but ties
    out["quant_rgb_fields"], out["quant_rgb_pixels"] = f3, fileio.image_from_fields(f3).pixels
    out["quant_gray_fields"], out["quant_gray_pixels"] = f1, fileio.image_from_fields(f1).pixels
    # P4 raster known answer, width not a multiple of 8
    m = rng.random((13, 21)) < 0.3
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "m.pbm")
        fileio.write_mask(path, m)
        raw = open(path, "rb").read()
        assert np.array_equal(fileio.read_mask(path), m)
    header = f"P4\n{m.shape[1]} {m.shape[0]}\n".encode()
    assert raw.startswith(header)
    out["raster_mask"] = m
    out["raster_bytes"] = np.frombuffer(raw[len(header):], dtype=np.uint8).reshape(m.shape[0], -1)
    # whole decodes
    for name, case in IMAGE_CASES.items():
        w, h, dens, seed, ch, bs, ov = case[:7]
        skw = case[7] if len(case) > 7 else {}
        prob = seeded(w, h, dens, seed, ch)
        px = prob.known.astype(np.uint8)
        image = fileio.ImageFile(px[0] if ch == 1 else np.moveaxis(px, 0, 2).copy())
        assert np.array_equal(image.channel_fields(), prob.known)
        cfg = dp.MultigridConfig(block_size=bs, overlap=ov, solver=dp.SolverConfig(**skw))
        res = dp.solve_image(dp.InpaintingProblem(prob.mask, image.channel_fields()), "mg-oras", cfg)
        out[f"{name}_pixels"] = fileio.image_from_fields(res.fields).pixels
        # distance of every value to the nearest rounding boundary: pixels closer than 1e-9 may differ
        out[f"{name}_margin_min"] = np.array(np.abs(res.fields - np.floor(res.fields) - 0.5).min())
        meta[name] = dict(w=w, h=h, density=dens, seed=seed, channels=ch, block_size=bs, overlap=ov, solver=skw,
                          iterations=[r.iterations for r in res.reports])
    np.savez_compressed(os.path.join(HERE, "golden_images.npz"), **out)
    with open(os.path.join(HERE, "golden_images.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print({k: v["iterations"] for k, v in meta.items()})


def kats():
    """Three known-answer tests of the reference's own suite, with the reference's outputs:
    TestBlockSolver.test_matches_scalar_local_solve (tests/test_solvers.py:156-169),
    TestVCycle.test_single_level_reduces_to_smoothing (tests/test_multigrid.py:218-233),
    TestFmgSolve.test_fine_unit_accounting (tests/test_multigrid.py:298-302)."""
    from diffpaint.partition import build_partition, build_weights
    out = {}
    # (a) batched block solve == scalar local solves, clamped blocks in both axes
    prob = seeded(80, 56, 0.15, 8)
    part = build_partition(80, 56, 32, 6)
    bs = sv.BlockSolver(prob.mask, 1.0, part, build_weights(part), alpha=0.5)
    r = np.random.default_rng(12345).normal(size=(56, 80))
    r[prob.mask] = 0.0
    target = 1e-5 * float(np.vdot(r, r))
    batched = bs.solve_blocks(bs.gather(r), target, max_iters=4096)
    for i, rect in enumerate(part.rects()):
        local = sv.build_local_system(rect, prob.mask, 1.0, 0.5)
        expected = sv.local_solve(local, r[rect.y0:rect.y0 + rect.h, rect.x0:rect.x0 + rect.w], target, 4096)
        np.testing.assert_allclose(batched[i], expected, atol=1e-12)
    out["kat_blocks_r"], out["kat_blocks_target"], out["kat_blocks_v"] = r, np.array(target), batched
    out["kat_blocks_scatter"] = bs.scatter_weighted(batched)
    # (b) a single-level V-cycle is nu_pre + nu_post Schwarz sweeps, bit for bit
    prob = seeded(32, 32, 0.1, 4)
    cfg = dp.MultigridConfig()
    hier = dp.build_hierarchy(prob, cfg)
    assert len(hier) == 1
    lev = hier.levels[0]
    u_cycle = prob.flat_init(0)
    mg.v_cycle(hier, 0, u_cycle, lev.rhs[0], cfg)
    u_manual = prob.flat_init(0)
    sv.oras_sweeps(lev.op, lev.block_solver(cfg.solver.alpha), lev.rhs[0], u_manual,
                   max_sweeps=cfg.nu_pre + cfg.nu_post, stop_norm=0.0, eta=cfg.solver.local_tol_fraction,
                   local_max_iters=4096)
    assert np.array_equal(u_cycle, u_manual)
    out["kat_vcycle_u"] = u_cycle
    # (c) fine-level work units = (nu_pre + nu_post) * cycles
    prob = seeded(128, 128, 0.05, 1)
    _, rep = dp.fmg_solve(dp.build_hierarchy(prob, cfg), cfg)
    assert rep.fine_smoother_iterations == (cfg.nu_pre + cfg.nu_post) * rep.iterations
    out["kat_units"] = np.array([rep.iterations, rep.fine_smoother_iterations])
    np.savez_compressed(os.path.join(HERE, "golden_kats.npz"), **out)
    print("kats:", out["kat_units"], batched.shape)


def anchors():
    os.environ["INPAINT_THREADS"] = "0"
    res = {}
    sample = {}
    for name, (w, h, dens, ch, bs, ov) in {
        "1080p_4pct_16_2": (1920, 1080, 0.04, 3, 16, 2),
        "4k_2pct_32_6": (3840, 2160, 0.02, 3, 32, 6),
        "4k_0.5pct_32_6": (3840, 2160, 0.005, 1, 32, 6),
    }.items():
        prob = seeded(w, h, dens, 0, ch)
        cfg = dp.MultigridConfig(block_size=bs, overlap=ov)
        r = dp.solve_image(prob, "mg-oras", cfg)
        res[name] = dict(w=w, h=h, density=dens, channels=ch, block_size=bs, overlap=ov, seed=0,
                         elapsed_s=r.elapsed, threads=os.cpu_count(),
                         reports=[dict(iterations=x.iterations, final_rel=x.final_rel_residual,
                                       baseline=x.baseline_residual, fine_units=x.fine_smoother_iterations,
                                       history=list(x.history)) for x in r.reports])
        sample[name] = r.fields.reshape(ch, -1)[:, ::997].copy()
        print(name, r.elapsed, [x.iterations for x in r.reports], flush=True)
    with open(os.path.join(HERE, "anchors.json"), "w") as f:
        json.dump(res, f, indent=1)
    np.savez_compressed(os.path.join(HERE, "anchors_sample.npz"), **sample)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--anchors", action="store_true")
    ap.add_argument("--pipelines", action="store_true", help="write only golden_pipelines.*")
    ap.add_argument("--images", action="store_true", help="write only golden_images.* (8-bit file path)")
    ap.add_argument("--kats", action="store_true", help="write only golden_kats.npz (reference-suite known answers)")
    a = ap.parse_args()
    if a.pipelines:
        pipelines()
    elif a.images:
        images()
    elif a.kats:
        kats()
    else:
        small()
        pipelines()
        images()
        kats()
        if a.anchors:
            anchors()
