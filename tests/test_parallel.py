"""Row-slab multi-GPU host logic (paper_2506_08793_b200/parallel.py)
on CPU: the slab driver's halo exchange (k*R rows every k sweeps), global stop rule
and gather run with torch.distributed over gloo (world sizes 1, 2 and 3), the
block engine being the oracle restatement applied to the extended slab (test
infrastructure).  The
restored field must equal the single-process oracle solve bit for bit (every
pixel's arithmetic is the same) and the residual norms to 1e-12 (only the
summation split differs)."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import TAU_STABLE
from oracle import pdz_oracle as orc
from paper_2506_08793_b200 import SolverConfig
from paper_2506_08793_b200.parallel import (SlabSolver, default_sweeps_per_exchange, halo_rows,
                                             slab_bounds, solve_slab)


# ---------------------------------------------------------------- oracle block

def oracle_block(settings, tau, edge=True):
    """Block engine for the CPU tests: n oracle sweeps (relaxed_step's
    arithmetic, separable Gaussian) of the extended slab as an image of its
    own, r^2 counted over rows [lo, hi)."""
    def block(u_ext, phi_e, lam_e, lo, hi, n):
        u = u_ext.numpy().copy()
        src, lam = phi_e.numpy(), lam_e.numpy()
        planes = u.shape[0]
        sums = np.zeros((n, planes))
        failed = np.zeros(planes, dtype=np.int32)
        for p in range(planes):
            for s in range(n):
                r = (orc.flux_divergence(u[p], settings.epsilon, edge)
                     - lam * orc.gaussian_blur_separable(u[p], settings.sigma,
                                                         settings.kernel_size) + src[p])
                u[p] = u[p] + tau * r
                sums[s, p] = np.sum(r[lo:hi] * r[lo:hi])
                if not failed[p] and not (np.all(np.isfinite(r[lo:hi]))
                                          and np.all(np.isfinite(u[p, lo:hi]))):
                    failed[p] = s + 1
        return torch.from_numpy(u), torch.from_numpy(sums), torch.from_numpy(failed)

    return block


# ------------------------------------------------------------------- inputs

def _problem(h=40, w=24, seed=3):
    rng = np.random.default_rng(seed)
    img = rng.uniform(0.1, 0.9, size=(h, w, 3))
    t = rng.uniform(0.3, 0.95, size=(h, w))
    a = np.array([0.9, 0.85, 0.8])
    st = orc.SolverSettings(tau=TAU_STABLE, sigma=1.5, kernel_size=7, max_iters=12,
                            rel_tol=1e-300)
    phi = np.stack([(img[:, :, c] - a[c] * (1.0 - t)) / np.maximum(t, st.t_floor)
                    for c in range(3)])
    lam = orc.haze_weight(t, st.lambda0, st.beta, st.lambda_monotonicity)
    return img, t, a, st, phi, lam


def _reference(img, t, a, st):
    outs, traces = [], []
    for c in range(3):
        u, tr = orc.relaxed_solve(img[:, :, c], t, float(a[c]), st, separable=True)
        outs.append(u)
        traces.append(tr)
    return np.stack(outs), traces


def _cfg(st, max_iters=None, rel_tol=None):
    return SolverConfig(tau=st.tau, sigma=st.sigma, kernel_size=st.kernel_size,
                        max_iters=max_iters or st.max_iters,
                        rel_tol=st.rel_tol if rel_tol is None else rel_tol)


# ------------------------------------------------------------------- tests

def test_slab_bounds_cover_the_image():
    for h, g in ((1024, 8), (4320, 8), (270, 3), (17, 4)):
        spans = [slab_bounds(h, g, k) for k in range(g)]
        assert spans[0][0] == 0 and spans[-1][1] == h
        assert all(spans[k][1] == spans[k + 1][0] for k in range(g - 1))
    assert slab_bounds(2160, 8, 3) == (810, 1080)  # C4 at G = 8: 270 rows each
    assert halo_rows(25) == 12 and halo_rows(49) == 24 and halo_rows(1) == 1
    with pytest.raises(ValueError):
        slab_bounds(10, 2, 2)
    # C4 at G = 8 (270 rows, R = 12): 4 sweeps per exchange; C5 (540, 24): 4
    assert default_sweeps_per_exchange(270, 12, 8, 500) == 4
    assert default_sweeps_per_exchange(30, 12, 8, 500) == 2
    assert default_sweeps_per_exchange(540, 24, 8, 3) == 3
    assert default_sweeps_per_exchange(10, 3, 1, 200) == 200


def test_slab_too_thin_for_the_halo():
    img, t, a, st, phi, lam = _problem(h=20)
    with pytest.raises(ValueError, match="halo"):
        SlabSolver(torch.from_numpy(phi), torch.from_numpy(lam), 20, _cfg(st), tau=st.tau,
                   rank=0, world=8, block=oracle_block(st, st.tau))
    with pytest.raises(ValueError, match="sweeps per exchange"):
        SlabSolver(torch.from_numpy(phi), torch.from_numpy(lam), 20, _cfg(st), tau=st.tau,
                   rank=0, world=2, block=oracle_block(st, st.tau), sweeps_per_exchange=4)


def test_single_slab_equals_the_oracle_bitwise():
    img, t, a, st, phi, lam = _problem()
    ref_u, ref_tr = _reference(img, t, a, st)
    u, traces = solve_slab(torch.from_numpy(phi), torch.from_numpy(lam), phi.shape[1], _cfg(st),
                           block=oracle_block(st, st.tau), warn=False)
    np.testing.assert_array_equal(u.numpy(), ref_u)
    for tr, rt in zip(traces, ref_tr):
        assert tr.residual_norms == rt.residual_norms
        assert tr.iterations_run == rt.iterations_run


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, outdir, max_iters, rel_tol, k):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        img, t, a, st, phi, lam = _problem()
        cfg = _cfg(st, max_iters, rel_tol)
        solver = SlabSolver(torch.from_numpy(phi), torch.from_numpy(lam), phi.shape[1], cfg,
                            tau=st.tau, rank=rank, world=world, block=oracle_block(st, st.tau),
                            sweeps_per_exchange=k)
        # halo exchange: the neighbour rows of the extended slab are replaced by
        # the neighbours' current rows (here: a marked copy of Phi)
        y0, y1, t, b = solver.y0, solver.y1, solver.top, solver.bot
        assert t == (0 if rank == 0 else k * solver.halo)
        assert b == (0 if rank == world - 1 else k * solver.halo)
        u = solver.u.clone()
        u[:, :t] = -1.0
        u[:, t + solver.rows:] = -1.0
        solver.exchange(u)
        np.testing.assert_array_equal(u.numpy(), phi[:, y0 - t:y1 + b])
        u_slab, traces = solve_slab(torch.from_numpy(phi), torch.from_numpy(lam), phi.shape[1],
                                    cfg, block=oracle_block(st, st.tau), sweeps_per_exchange=k,
                                    warn=False)
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), u=u_slab.numpy(), y0=y0, y1=y1,
                 **{f"norms{c}": np.array(tr.residual_norms) for c, tr in enumerate(traces)},
                 iters=np.array([tr.iterations_run for tr in traces]),
                 conv=np.array([tr.converged for tr in traces]))
    finally:
        dist.destroy_process_group()


def _run_world(world, max_iters=12, rel_tol=1e-300, k=2):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d, max_iters, rel_tol, k), nprocs=world,
                 join=True)
        return [np.load(os.path.join(d, f"rank{k}.npz"), allow_pickle=True)
                for k in range(world)]


@pytest.mark.parametrize("world,k", [(2, 1), (2, 3), (3, 2), (3, 4)])
def test_row_slabs_over_gloo_match_the_oracle(world, k):
    # 12 sweeps in blocks of k (the last block shorter when k does not divide 12)
    img, t, a, st, phi, lam = _problem()
    ref_u, ref_tr = _reference(img, t, a, st)
    parts = _run_world(world, k=k)
    u = np.concatenate([p["u"] for p in parts], axis=1)
    np.testing.assert_array_equal(u, ref_u)
    for p in parts:  # every rank holds the same global trace
        for c in range(3):
            np.testing.assert_allclose(p[f"norms{c}"], ref_tr[c].residual_norms, rtol=1e-12)
            assert int(p["iters"][c]) == ref_tr[c].iterations_run


def test_row_slabs_share_the_global_stop_rule():
    img, t, a, st, phi, lam = _problem()
    st_tol = orc.SolverSettings(tau=st.tau, sigma=st.sigma, kernel_size=st.kernel_size,
                                max_iters=200, rel_tol=2e-3)
    ref_u, ref_tr = _reference(img, t, a, st_tol)
    assert all(tr.converged for tr in ref_tr) and ref_tr[0].iterations_run < 200
    # blocks of 3 sweeps: planes stop inside blocks and take the recomputed
    # iterate after their stopping sweep
    parts = _run_world(2, max_iters=200, rel_tol=2e-3, k=3)
    u = np.concatenate([p["u"] for p in parts], axis=1)
    for c in range(3):
        assert [int(p["iters"][c]) for p in parts] == [ref_tr[c].iterations_run] * 2
        assert all(bool(p["conv"][c]) for p in parts)
    np.testing.assert_array_equal(u, ref_u)


def _gather_worker(rank, world, port, outdir, height):
    from paper_2506_08793_b200.parallel import _all_gather_rows

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = torch.arange(3 * height * 5, dtype=torch.float32).reshape(3, height, 5)
        y0, y1 = slab_bounds(height, world, rank)
        out = _all_gather_rows(full[:, y0:y1].contiguous(), height, None, rank, world)
        np.save(os.path.join(outdir, f"g{rank}.npy"), out.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,height", [(2, 9), (3, 10), (3, 7)])
def test_all_gather_rows_over_gloo(world, height):
    """The final slab gather of dehaze_slabs: ragged last slab (ceil(H/G)
    rows per rank, remainder on the last), every rank gets the full field."""
    full = np.arange(3 * height * 5, dtype=np.float32).reshape(3, height, 5)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_gather_worker, args=(world, _free_port(), d, height), nprocs=world, join=True)
        for r in range(world):
            np.testing.assert_array_equal(np.load(os.path.join(d, f"g{r}.npy")), full)
