"""Row-slab multi-GPU host logic (paper_2506_08793_b200/parallel.py)
on CPU: the slab driver's halo exchange, global stop rule and gather run with
torch.distributed over gloo (world size 1 and 2), the sweep itself being the
oracle restatement applied to the extended slab (test infrastructure).  The
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
from paper_2506_08793_b200.parallel import SlabSolver, halo_rows, slab_bounds, solve_slab


# ---------------------------------------------------------------- oracle step

def _gy_global(u, y_off, height):
    """np.gradient along rows of the extended slab with the one-sided ends
    only at global rows 0 / H-1 (there the reflected halo row equals the edge
    row, so u[i+1] - u[i-1] is exactly np.gradient's one-sided difference)."""
    g = np.empty_like(u)
    g[1:-1] = (u[2:] - u[:-2]) / 2.0
    g[0] = u[1] - u[0]
    g[-1] = u[-1] - u[-2]
    for i in range(1, u.shape[0] - 1):
        if i + y_off in (0, height - 1):
            g[i] = u[i + 1] - u[i - 1]
    return g


def _slab_divergence(u, eps, edge, y_off, height):
    je = u[:, 1:] - u[:, :-1]
    js = u[1:, :] - u[:-1, :]
    if edge:
        gy = _gy_global(u, y_off, height)
        gx = orc._centred(u, 1)
        te = 0.5 * (gy[:, 1:] + gy[:, :-1])
        ts = 0.5 * (gx[1:, :] + gx[:-1, :])
        de = 1.0 / (np.sqrt(je * je + te * te) + eps)
        ds = 1.0 / (np.sqrt(js * js + ts * ts) + eps)
    else:
        de, ds = np.ones_like(je), np.ones_like(js)
    fe, fs = de * je, ds * js
    acc = np.zeros_like(u)
    acc[:, :-1] = acc[:, :-1] + fe
    acc[:, 1:] = acc[:, 1:] - fe
    acc[:-1, :] = acc[:-1, :] + fs
    acc[1:, :] = acc[1:, :] - fs
    return acc


def _slab_blur(u, sigma, size, lo, hi):
    """gaussian_blur_separable restricted to rows [lo, hi) of the slab; the
    R rows above / below come from the halo instead of reflection."""
    h, w = u.shape
    r = size // 2
    g = orc.gaussian_taps_1d(sigma, size)
    cols = orc.reflect_index(np.arange(-r, w + r), w)
    ext = u[:, cols]
    tmp = np.zeros_like(u)
    for b in range(size):
        tmp += g[b] * ext[:, b:b + w]
    out = np.zeros((hi - lo, w))
    for a in range(size):
        out += g[a] * tmp[lo - r + a:hi - r + a, :]
    return out


def oracle_slab_step(settings, tau, edge=True):
    def step(u_in, u_out, phi_e, lam_e, y_off, height, lo, hi):
        u = u_in.numpy()
        src, lam = phi_e.numpy(), lam_e.numpy()
        out = u_out.numpy()
        planes = u.shape[0]
        sums = np.zeros(planes)
        nf = np.zeros(planes, dtype=np.int32)
        for p in range(planes):
            div = _slab_divergence(u[p], settings.epsilon, edge, y_off, height)[lo:hi]
            r = div - lam[lo:hi] * _slab_blur(u[p], settings.sigma, settings.kernel_size,
                                              lo, hi) + src[p, lo:hi]
            out[p, lo:hi] = u[p, lo:hi] + tau * r
            sums[p] = np.sum(r * r)
            nf[p] = int(not (np.all(np.isfinite(r)) and np.all(np.isfinite(out[p, lo:hi]))))
        return torch.from_numpy(sums), torch.from_numpy(nf)

    return step


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


def test_slab_too_thin_for_the_halo():
    img, t, a, st, phi, lam = _problem(h=20)
    with pytest.raises(ValueError, match="halo"):
        SlabSolver(torch.from_numpy(phi), torch.from_numpy(lam), 20, _cfg(st), tau=st.tau,
                   rank=0, world=8, step=oracle_slab_step(st, st.tau))


def test_single_slab_equals_the_oracle_bitwise():
    img, t, a, st, phi, lam = _problem()
    ref_u, ref_tr = _reference(img, t, a, st)
    u, traces = solve_slab(torch.from_numpy(phi), torch.from_numpy(lam), phi.shape[1], _cfg(st),
                           step=oracle_slab_step(st, st.tau), warn=False)
    np.testing.assert_array_equal(u.numpy(), ref_u)
    for tr, rt in zip(traces, ref_tr):
        assert tr.residual_norms == rt.residual_norms
        assert tr.iterations_run == rt.iterations_run


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, outdir, max_iters, rel_tol):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        img, t, a, st, phi, lam = _problem()
        cfg = _cfg(st, max_iters, rel_tol)
        solver = SlabSolver(torch.from_numpy(phi), torch.from_numpy(lam), phi.shape[1], cfg,
                            tau=st.tau, rank=rank, world=world, step=oracle_slab_step(st, st.tau))
        # halo exchange: after one exchange the halos hold the neighbours' rows
        u = solver.u[0].clone()
        solver.exchange(u)
        R, n = solver.halo, solver.rows
        y0, y1 = solver.y0, solver.y1
        rows = orc.reflect_index(np.arange(y0 - R, y1 + R), phi.shape[1])
        np.testing.assert_array_equal(u.numpy(), phi[:, rows])
        u_slab, traces = solve_slab(torch.from_numpy(phi), torch.from_numpy(lam), phi.shape[1],
                                    cfg, step=oracle_slab_step(st, st.tau), warn=False)
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), u=u_slab.numpy(), y0=y0, y1=y1,
                 **{f"norms{c}": np.array(tr.residual_norms) for c, tr in enumerate(traces)},
                 iters=np.array([tr.iterations_run for tr in traces]),
                 conv=np.array([tr.converged for tr in traces]))
    finally:
        dist.destroy_process_group()


def _run_world(world, max_iters=12, rel_tol=1e-300):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d, max_iters, rel_tol), nprocs=world,
                 join=True)
        return [np.load(os.path.join(d, f"rank{k}.npz"), allow_pickle=True)
                for k in range(world)]


@pytest.mark.parametrize("world", [2, 3])
def test_row_slabs_over_gloo_match_the_oracle(world):
    img, t, a, st, phi, lam = _problem()
    ref_u, ref_tr = _reference(img, t, a, st)
    parts = _run_world(world)
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
    parts = _run_world(2, max_iters=200, rel_tol=2e-3)
    u = np.concatenate([p["u"] for p in parts], axis=1)
    for c in range(3):
        assert [int(p["iters"][c]) for p in parts] == [ref_tr[c].iterations_run] * 2
        assert all(bool(p["conv"][c]) for p in parts)
    np.testing.assert_array_equal(u, ref_u)
