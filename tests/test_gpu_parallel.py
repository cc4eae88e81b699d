"""Row-slab sweep on the GPU (pdz_fixed_point_step_rows; parallel.py).

One GPU only: each slab's halo is filled from the whole field exactly as the
neighbouring ranks would send it, so the slab sweep must reproduce the
whole-image sweep's rows bit for bit (same kernel arithmetic, global-row
np.gradient ends).  The single-rank slab driver must track the persistent
solve and the oracle."""

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
