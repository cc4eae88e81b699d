"""Row-slab mode on the GPU (pdz_fixed_point_step_rows,
pdz_fixed_point_sweeps_from; parallel.py).

One GPU only: each slab's halo is filled from the whole field exactly as the
neighbouring ranks would send it, so the slab sweep must reproduce the
whole-image sweep's rows bit for bit (same kernel arithmetic, global-row
np.gradient ends).  The blocked slab driver runs G emulated ranks as threads
of one process (an in-process exchange / all-reduce stands in for NCCL; the
ranks' kernels never wait on each other) and must track the whole-image
persistent solve and the oracle."""

import threading

import numpy as np
import pytest
import torch

from conftest import TAU_STABLE
from oracle import pdz_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pdz():
    import paper_2506_08793_b200 as p

    return p


def _fields(h, w, c, seed=5):
    rng = np.random.default_rng(seed)
    u = rng.uniform(0.0, 1.0, size=(c, h, w)).astype(np.float32)
    phi = rng.uniform(-0.2, 1.2, size=(c, h, w)).astype(np.float32)
    lam = rng.uniform(0.02, 0.5, size=(h, w)).astype(np.float32)
    return u, phi, lam


@pytest.mark.parametrize("k,edge", [(19, 1), (13, 1), (5, 0), (1, 1)])
def test_step_rows_equals_whole_image_sweep(pdz, k, edge):
    from paper_2506_08793_b200 import _native as nat
    from paper_2506_08793_b200.solver import _params

    h, w, c = 70, 96, 3
    u, phi, lam = _fields(h, w, c)
    cfg = pdz.SolverConfig(tau=TAU_STABLE, sigma=3.0, kernel_size=k)
    lib = nat.lib()
    dev = torch.device("cuda")
    U, PH, LM = (torch.from_numpy(x).to(dev) for x in (u, phi, lam))
    prm = _params(h, w, c, c, cfg, edge_preserving=bool(edge), tau=TAU_STABLE)
    ws = torch.empty(lib.pdz_step_workspace_bytes(prm), dtype=torch.uint8, device=dev)
    full = torch.empty_like(U)
    norms = torch.empty(c, dtype=torch.float64, device=dev)
    nat.check(lib.pdz_fixed_point_step(prm, nat.ptr(U), nat.ptr(full), nat.ptr(PH), nat.ptr(LM),
                                       nat.ptr(norms), None, nat.ptr(ws), ws.numel(),
                                       nat.stream_ptr()))
    R = max(1, k // 2)
    total = torch.zeros(c, dtype=torch.float64, device=dev)
    for y0, y1 in ((0, 20), (20, 45), (45, 70)):
        rows = orc.reflect_index(np.arange(y0 - R, y1 + R), h)
        ue = U[:, torch.from_numpy(rows).to(dev)].contiguous()
        pe = PH[:, torch.from_numpy(rows).to(dev)].contiguous()
        le = LM[torch.from_numpy(rows).to(dev)].contiguous()
        E = y1 - y0 + 2 * R
        prm_e = _params(E, w, c, c, cfg, edge_preserving=bool(edge), tau=TAU_STABLE)
        ws_e = torch.empty(lib.pdz_step_workspace_bytes(prm_e), dtype=torch.uint8, device=dev)
        out = torch.zeros_like(ue)
        sums = torch.empty(c, dtype=torch.float64, device=dev)
        nf = torch.empty(c, dtype=torch.int32, device=dev)
        nat.check(lib.pdz_fixed_point_step_rows(
            prm_e, nat.ptr(ue), nat.ptr(out), nat.ptr(pe), nat.ptr(le), y0 - R, h, R, R + y1 - y0,
            nat.ptr(sums), nat.ptr(nf), nat.ptr(ws_e), ws_e.numel(), nat.stream_ptr()))
        torch.testing.assert_close(out[:, R:R + y1 - y0], full[:, y0:y1], rtol=0, atol=0)
        assert int(nf.max()) == 0
        total += sums
    torch.testing.assert_close(total.sqrt(), norms, rtol=1e-12, atol=0)


def test_step_rows_validates_the_window(pdz):
    from paper_2506_08793_b200 import _native as nat
    from paper_2506_08793_b200.solver import _params

    lib = nat.lib()
    cfg = pdz.SolverConfig(kernel_size=5)
    prm = _params(10, 8, 1, 1, cfg)
    buf = torch.zeros((10, 8), device="cuda")
    sums = torch.zeros(1, dtype=torch.float64, device="cuda")
    ws = torch.empty(lib.pdz_step_workspace_bytes(prm), dtype=torch.uint8, device="cuda")
    args = (nat.ptr(buf), nat.ptr(torch.empty_like(buf)), nat.ptr(buf), nat.ptr(buf))
    rc = lib.pdz_fixed_point_step_rows(prm, *args, 0, 10, 0, 10, nat.ptr(sums), None,
                                       nat.ptr(ws), ws.numel(), nat.stream_ptr())
    assert rc == nat.PDZ_EINVAL  # no halo row
    rc = lib.pdz_fixed_point_step_rows(prm, *args, 5, 10, 2, 8, nat.ptr(sums), None,
                                       nat.ptr(ws), ws.numel(), nat.stream_ptr())
    assert rc == nat.PDZ_EINVAL  # window beyond the image


def test_single_rank_slab_solve_tracks_the_persistent_solve(pdz):
    from paper_2506_08793_b200.parallel import solve_slab
    from paper_2506_08793_b200.solver import DeviceProblem, solve_problem

    h, w, c = 96, 128, 3
    _, phi, lam = _fields(h, w, c, seed=9)
    cfg = pdz.SolverConfig(tau=TAU_STABLE, sigma=3.0, kernel_size=19, max_iters=40,
                           rel_tol=1e-300)
    PH = torch.from_numpy(phi).cuda()
    LM = torch.from_numpy(lam).cuda()
    u_slab, tr_slab = solve_slab(PH, LM, h, cfg, warn=False)
    u_ref, tr_ref = solve_problem(DeviceProblem(PH, LM, h, w, c, c, np.ones(c)), cfg, warn=False)
    assert float((u_slab - u_ref).abs().max()) <= 1e-5
    for a, b in zip(tr_slab, tr_ref):
        assert a.iterations_run == b.iterations_run == 40
        np.testing.assert_allclose(a.residual_norms, b.residual_norms, rtol=1e-5)


class _ThreadRanks:
    """In-process stand-in for torch.distributed between G SlabSolvers run in
    threads: the same rows travel as the NCCL point-to-point exchange would
    send them, and the all-reduce sums the ranks' tables in rank order."""

    def __init__(self, world):
        self.world = world
        self.bar = threading.Barrier(world)
        self.slot = {}

    def attach(self, solver):
        group = self

        def exchange(u):
            t, n, b = solver.top, solver.rows, solver.bot
            group.slot[solver.rank] = (u[:, t:t + n].clone(),)
            group.bar.wait()
            if t:
                u[:, :t] = group.slot[solver.rank - 1][0][:, -t:]
            if b:
                u[:, t + n:] = group.slot[solver.rank + 1][0][:, :b]
            group.bar.wait()

        def allreduce(sums, failed):
            group.slot[solver.rank] = (sums, failed)
            group.bar.wait()
            tot = sum(group.slot[r][0] for r in range(group.world))
            fl = torch.stack([group.slot[r][1] for r in range(group.world)])
            fl = torch.where(fl > 0, fl, torch.full_like(fl, 1 << 30)).min(dim=0).values
            fl = torch.where(fl == (1 << 30), torch.zeros_like(fl), fl)
            group.bar.wait()
            return tot, fl

        solver.exchange = exchange
        solver._allreduce = allreduce
        return solver


def _emulated_slabs(pdz, phi, lam, h, cfg, world, k):
    from paper_2506_08793_b200.parallel import SlabSolver

    group = _ThreadRanks(world)
    out = [None] * world
    errs = []

    def run(rank):
        try:
            sv = group.attach(SlabSolver(phi, lam, h, cfg, tau=cfg.tau, rank=rank, world=world,
                                         sweeps_per_exchange=k))
            out[rank] = sv.solve(cfg.max_iters, cfg.rel_tol)
        except Exception as e:  # noqa: BLE001 - re-raised in the main thread
            errs.append(e)
            group.bar.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("h,w,ksz,world,k", [(600, 256, 13, 3, 4), (520, 192, 25, 4, 3),
                                             (400, 128, 49, 2, 2), (300, 136, 19, 3, 1)])
def test_blocked_slabs_track_the_whole_image_solve(pdz, h, w, ksz, world, k):
    from paper_2506_08793_b200.solver import DeviceProblem, solve_problem

    c = 3
    _, phi, lam = _fields(h, w, c, seed=ksz)
    cfg = pdz.SolverConfig(tau=TAU_STABLE, sigma=ksz / 6.0, kernel_size=ksz, max_iters=14,
                           rel_tol=1e-300)
    PH = torch.from_numpy(phi).cuda()
    LM = torch.from_numpy(lam).cuda()
    parts = _emulated_slabs(pdz, PH, LM, h, cfg, world, k)
    u = torch.cat([p[0] for p in parts], dim=1)
    u_ref, tr_ref = solve_problem(DeviceProblem(PH, LM, h, w, c, c, np.ones(c)), cfg, warn=False)
    assert float((u - u_ref).abs().max()) <= 1e-6
    for p in parts:  # every rank holds the global trace
        for ch in range(c):
            assert p[2][ch] == tr_ref[ch].iterations_run == 14
            np.testing.assert_allclose(p[1][ch], tr_ref[ch].residual_norms, rtol=1e-6)
    st = orc.SolverSettings.from_config(cfg)
    for ch in range(c):
        ru = phi[ch].astype(np.float64)
        src, lm = phi[ch].astype(np.float64), lam.astype(np.float64)
        for _ in range(cfg.max_iters):
            ru, _ = orc.relaxed_step(ru, src, lm, st, separable=True)
        assert np.max(np.abs(u[ch].cpu().numpy() - ru)) <= 1e-4


def test_blocked_slabs_stop_inside_a_block(pdz):
    # planes stop at different sweeps inside 4-sweep blocks: each takes the
    # iterate after its own stopping sweep, like the whole-image solve
    from paper_2506_08793_b200.solver import DeviceProblem, solve_problem

    h, w, c = 360, 128, 3
    _, phi, lam = _fields(h, w, c, seed=21)
    cfg = pdz.SolverConfig(tau=TAU_STABLE, sigma=2.0, kernel_size=13, max_iters=400,
                           rel_tol=3e-3)
    PH = torch.from_numpy(phi).cuda()
    LM = torch.from_numpy(lam).cuda()
    u_ref, tr_ref = solve_problem(DeviceProblem(PH, LM, h, w, c, c, np.ones(c)), cfg, warn=False)
    runs = [tr.iterations_run for tr in tr_ref]
    assert all(tr.converged for tr in tr_ref) and max(runs) < 400
    parts = _emulated_slabs(pdz, PH, LM, h, cfg, 3, 4)
    u = torch.cat([p[0] for p in parts], dim=1)
    for p in parts:
        assert p[2] == runs and all(p[3])
    assert float((u - u_ref).abs().max()) <= 1e-6
