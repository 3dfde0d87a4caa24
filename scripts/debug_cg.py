import sys; sys.path.insert(0, '.')
import numpy as np, oracle
import paper_2401_06744_b200 as bp
w, h, d, s, bs, ov = 96, 64, 0.10, 1, 16, 2
m, k = oracle.seeded_problem(w, h, d, s, channels=1)
for name in ("cg", "ml-cg", "mg-cg"):
    cfg_b = bp.MultigridConfig(block_size=bs, overlap=ov)
    res = bp.solve_image(bp.InpaintingProblem(m, k), name, cfg_b)
    if name == "cg":
        ref, ro = oracle.cg_solve(m, k[0], 1.0, oracle.SolverConfig())
    else:
        mode = "multilevel" if name.startswith("ml") else "full_multigrid"
        refs, reps = oracle.solve_image(m, k, 1.0, oracle.MultigridConfig(block_size=bs, overlap=ov, smoother="cg", mode=mode))
        ref, ro = refs[0], reps[0]
    rg = res.reports[0]
    print(name, "gpu", rg.iterations, rg.fine_smoother_iterations, rg.final_rel_residual, rg.history[:6])
    print(name, "orc", ro.iterations, ro.fine_smoother_iterations, ro.final_rel_residual, ro.history[:6], np.abs(res.fields[0] - ref).max())
