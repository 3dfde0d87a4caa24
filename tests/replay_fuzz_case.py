"""Test helper (not collected): replays one case of test_randomised_shapes_and_configs_match_oracle
(python tests/replay_fuzz_case.py SEED CASE) and prints the histories of the oracle and of the CUDA path."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_2401_06744_b200 as bp
seed, target = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(seed)
geoms = [(32, 6), (16, 2), (8, 2), (24, 4), (32, 0), (16, 8), (10, 3), (40, 6), (64, 6)]
for case in range(target + 1):
    w, h = int(rng.integers(9, 260)), int(rng.integers(9, 200))
    if case % 5 == 0:
        w, h = 4 * (w // 4 + 1), 2 * (h // 2 + 1)
    bs, ov = geoms[int(rng.integers(len(geoms)))]
    dens = float(rng.choice([0.01, 0.03, 0.1, 0.3, 0.8]))
    dens = max(dens, 2.0 / (w * h))
    c = int(rng.integers(1, 4))
    kw = dict(tol_rel=float(rng.choice([1e-3, 1e-5])), alpha=float(rng.choice([0.5, 1.0, 0.2])))
    mkw = dict(nu_pre=int(rng.integers(0, 3)), nu_post=int(rng.integers(1, 3)),
               value_downsampling=str(rng.choice(["modified", "naive"])))
    spacing_case = (w, h, bs, ov, dens, c, kw, mkw)
    m, k = (None, None)
    spacing = float(rng.choice([1.0, 0.5, 2.0]))
print(spacing_case, spacing)
m, k = oracle.seeded_problem(w, h, dens, 500 + target, channels=c)
cfg_o = oracle.MultigridConfig(block_size=bs, overlap=ov, solver=oracle.SolverConfig(**kw), **mkw)
cfg_b = bp.MultigridConfig(block_size=bs, overlap=ov, solver=bp.SolverConfig(**kw), **mkw)
ref, ro = oracle.solve_image(m, k, spacing, cfg_o)
res = bp.solve_image(bp.InpaintingProblem(m, k, spacing), "mg-oras", cfg_b)
for a, b in zip(ro, res.reports):
    print("cycles", a.iterations, b.iterations, "units", a.fine_smoother_iterations, b.fine_smoother_iterations)
    for i, (x, y) in enumerate(zip(a.history, b.history)):
        print(f"  {i:3d} {x:.12e} {y:.12e} {abs(x - y) / x:.2e}")
print("max abs field diff", np.abs(ref - res.fields).max())
