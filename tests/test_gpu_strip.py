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


def _run_virtual(nranks, w, h, c, cfg, mask, known, levels=1):
    group = strip.LocalGroup(nranks)
    out, errs = [None] * nranks, []

    def work(r):
        try:
            s = strip.StripSolver(w, h, c, cfg, group.transport(r), levels=levels)
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


@pytest.mark.parametrize("w,h,dens,seed,nranks,levels", [
    (640, 400, 0.02, 3, 2, 1),
    (640, 400, 0.02, 3, 3, 1),
    (512, 700, 0.05, 5, 4, 1),      # clamped last block row, uneven strips
    (1920, 1080, 0.04, 0, 4, 1),
    (3840, 2160, 0.02, 0, 8, 1),    # the 8-GPU layout of BASELINE config 4 at 4K
    (640, 400, 0.02, 3, 2, 2),      # two striped levels: halo exchange of the restricted residual too
    (1920, 1080, 0.04, 0, 4, 2),
    (3840, 2160, 0.02, 0, 8, 2),
    (3840, 2160, 0.02, 0, 4, 3),
])
def test_strip_solve_matches_single_plan(w, h, dens, seed, nranks, levels):
    c = 2
    m, k = oracle.seeded_problem(w, h, dens, seed, channels=c)
    cfg = bp.MultigridConfig(block_size=32, overlap=6)
    ref = bp.solve_image(bp.InpaintingProblem(m, k), "mg-oras", cfg)
    parts = _run_virtual(nranks, w, h, c, cfg, m, k, levels)
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
    n = 8
    ranges = strip.strip_ranges(2160, 32, 6, n)
    assert ranges[0][0] == 0 and ranges[-1][1] == 2160
    for a, b in zip(ranges, ranges[1:]):
        assert a[1] == b[0]                      # strips tile the image
        assert b[4] <= a[5] - 1                  # the boundary block row is solved on both sides
    for own_lo, own_hi, ext_lo, ext_hi, iy_lo, iy_hi in ranges:
        assert own_lo % 2 == 0 and ext_lo % 2 == 0 and ext_lo <= max(0, own_lo - 1) and ext_hi >= min(2160, own_hi + 1)
        assert ext_hi - own_hi <= 34 + 26 and own_lo - ext_lo <= 28 + 26   # one-block-deep halos
    # what rank 3 receives is exactly what its neighbours send to it
    recv, _ = strip.halo_plan(ranges, 3)
    sends = []
    for q in range(n):
        if q != 3:
            sends += [(q, a, b) for (dst, a, b) in strip.halo_plan(ranges, q)[1] if dst == 3]
    assert sorted(recv) == sorted(sends)
    rows = strip.coarse_rows(ranges, 1080)
    assert rows[0][0] == 0 and rows[-1][1] == 1080 and all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
    # two striped levels: the cuts halve exactly, the level-1 halo covers what level 0's prolongation reads
    r2 = strip.strip_ranges(2160, 32, 6, n, levels=2)
    for q in range(n):
        l0, l1 = r2[0][q], r2[1][q]
        assert l1[0] == l0[0] // 2 and (l1[1] == l0[1] // 2 or q == n - 1)
        assert l1[2] <= max(0, l0[2] // 2 - 1) and l1[3] >= min(1080, (l0[3] + 1) // 2 + 1)


# ---- two real PROCESSES on the one GPU: peer memory through CUDA IPC, control through gloo ----------

def _ipc_worker(rank, world, port, w, h, c, levels, q):
    import os
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m, k = oracle.seeded_problem(w, h, 0.03, 7, channels=c)
    s = strip.StripSolver(w, h, c, bp.MultigridConfig(), strip.IpcTransport(), levels=levels)
    u, reps = s.solve(m, k)
    q.put((rank, s.own, u.cpu().numpy(), [(r.iterations, r.final_rel_residual) for r in reps]))
    dist.barrier()
    s.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,levels", [(2, 1), (3, 2)])
def test_strip_solve_over_cuda_ipc_processes(world, levels):
    """One process per rank (all on this GPU), buffers mapped into each other with CUDA IPC, halo rows
    pulled with device-to-device copies: the multi-process shape of the multi-GPU run."""
    import socket
    import torch.multiprocessing as mp
    w, h, c = 768, 512, 2
    m, k = oracle.seeded_problem(w, h, 0.03, 7, channels=c)
    ref = bp.solve_image(bp.InpaintingProblem(m, k), "mg-oras", bp.MultigridConfig())
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, w, h, c, levels, q)) for r in range(world)]
    for p in procs:
        p.start()
    full = np.empty_like(ref.fields)
    for _ in range(world):
        rank, (lo, hi), u, reps = q.get(timeout=300)
        full[:, lo:hi] = u
        assert [it for it, _ in reps] == [r.iterations for r in ref.reports]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    np.testing.assert_allclose(full, ref.fields, rtol=0, atol=1e-9)


def test_native_nccl_strip_one_rank_runs_as_graphs():
    """b200p_plan_set_strip_nccl: the library issues the exchanges itself (ncclAllReduce of the partial norms on a
    one-rank communicator here; halo send / recv have no peer) and the strip solve is captured as graphs.  Same
    cycle counts and fields as the whole-image plan; the second solve (graph replay) equals the first (eager
    warm-up) bit for bit."""
    w, h, c = 640, 400, 3
    m, k = oracle.seeded_problem(w, h, 0.02, 3, channels=c)
    cfg = bp.MultigridConfig(block_size=32, overlap=6, solver=bp.SolverConfig(tol_rel=1e-6))
    ref = bp.solve_image(bp.InpaintingProblem(m, k), "mg-oras", cfg)
    for levels in (1, 2):
        t = strip.NcclNative()
        assert (t.rank, t.nranks) == (0, 1)
        s = strip.StripSolver(w, h, c, cfg, t, levels=levels)
        out1, reps1 = s.solve(m, k)
        out1 = out1.cpu().numpy()
        launches = s.plan.launch_count
        out2, reps2 = s.solve(m, k)
        out2 = out2.cpu().numpy()
        assert s.plan.launch_count > launches
        assert [r.iterations for r in reps1] == [r.iterations for r in reps2] == [r.iterations for r in ref.reports]
        assert np.array_equal(out1, out2)
        assert np.abs(out1 - ref.fields).max() <= 1e-9
        for r1, r0 in zip(reps2, ref.reports):
            assert r1.final_rel_residual == pytest.approx(r0.final_rel_residual, rel=1e-9)
        s.close()
    with pytest.raises(ValueError, match="communicator is rank"):
        t = strip.NcclNative()
        plan = bp.Plan(w, h, c, 1, cfg)
        rg = strip.strip_ranges(h, 32, 6, 2, 1)
        flat = [v for q in range(2) for v in rg[q]]
        import ctypes as C
        from paper_2401_06744_b200 import _lib
        arr = (C.c_int * len(flat))(*flat)
        try:
            _lib.check(_lib.lib().b200p_plan_set_strip_nccl(plan.handle, 1, C.cast(arr, C.c_void_p), 0, 2, t.comm))
        finally:
            plan.close()
            t.close()
