"""Small solves that walk every sync protocol of the persistent kernel, for
compute-sanitizer (one tool per run; profiles/r2_sanitizer_*.txt):

    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_cases.py

Cases: a partial last strip (W % 64 != 0: the shared-memory pad reflection
behind both TMA boxes), K = 49 (R = 24, the 95-row geometry), the stop rule
with planes stopping at different sweeps (finaliser CTA, frozen planes), a
batch (CTA ranges over several images), a multi-block pass (geometry V = 1)
and one row-slab block from a resident iterate.  Every result is checked
against the CPU oracle (max-abs 1e-4), so a tool-induced timeout or a wrong
answer fails loudly."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2506_08793_b200 as pdz  # noqa: E402
from oracle import pdz_oracle as orc  # noqa: E402

TAU = 0.9 * 2.0 / (8.0 / 1e-3 + 0.5)


def fields(h, w, seed):
    rng = np.random.default_rng(seed)
    ch = rng.random((h, w)) * 0.8 + 0.1
    t = 0.3 + 0.6 * rng.random((h, w))
    return ch, t


def solve_case(name, h, w, k, iters, rel_tol=1e-300, env=None):
    for key, val in (env or {}).items():
        os.environ[key] = val
    ch, t = fields(h, w, h + w + k)
    cfg = pdz.SolverConfig(tau=TAU, kernel_size=k, sigma=max(1.0, k / 6.0), max_iters=iters,
                           rel_tol=rel_tol)
    u, tr = pdz.fixed_point_solve(ch, t, 0.9, cfg)
    ru, rtr = orc.relaxed_solve(ch, t, 0.9, orc.SolverSettings.from_config(cfg), separable=True)
    err = float(np.max(np.abs(u - ru)))
    for key in (env or {}):
        del os.environ[key]
    ok = err <= 1e-4 and tr.iterations_run == rtr.iterations_run
    print(f"{name}: {h}x{w} K={k} sweeps={tr.iterations_run} max-abs {err:.2e} "
          f"{'ok' if ok else 'MISMATCH'}", flush=True)
    return ok


def batch_case():
    rng = np.random.default_rng(5)
    imgs = [rng.random((64, 128, 3)) * 0.8 + 0.1 for _ in range(3)]
    cfg = pdz.SolverConfig(tau=TAU, kernel_size=5, sigma=1.0, patch_radius=2, max_iters=6,
                           rel_tol=3e-2)
    flags = ("no-multiscale", "no-guided")
    out, res = pdz.dehaze_batch(imgs, cfg, ablation=flags)
    ok = True
    for i, im in enumerate(imgs):
        ro, _, _, rtr = orc.run_pipeline(im, orc.SolverSettings.from_config(cfg), flags,
                                         separable=True)
        err = float(np.max(np.abs(out[i] - ro)))
        same = [a.iterations_run for a in res[i].traces] == [b.iterations_run for b in rtr]
        ok &= err <= 1e-4 and same
    print(f"batch: 3 x 64x128x3 K=5 stop rule {'ok' if ok else 'MISMATCH'}", flush=True)
    return ok


def slab_case():
    import torch

    from paper_2506_08793_b200.parallel import solve_slab
    from paper_2506_08793_b200.solver import DeviceProblem, solve_problem

    rng = np.random.default_rng(11)
    phi = torch.from_numpy(rng.uniform(0.0, 1.0, (2, 96, 128)).astype(np.float32)).cuda()
    lam = torch.from_numpy(rng.uniform(0.05, 0.5, (96, 128)).astype(np.float32)).cuda()
    cfg = pdz.SolverConfig(tau=TAU, kernel_size=7, sigma=1.5, max_iters=7, rel_tol=1e-300)
    u, _ = solve_slab(phi, lam, 96, cfg, warn=False, sweeps_per_exchange=3)
    ref, _ = solve_problem(DeviceProblem(phi, lam, 96, 128, 2, 2, np.ones(2)), cfg, warn=False)
    err = float((u - ref).abs().max())
    print(f"slab (resident blocks of 3 sweeps): max-abs vs whole solve {err:.2e} "
          f"{'ok' if err <= 1e-6 else 'MISMATCH'}", flush=True)
    return err <= 1e-6


def main():
    ok = True
    ok &= solve_case("partial strip", 96, 136, 13, 4)
    ok &= solve_case("K=49", 120, 128, 49, 3)
    ok &= solve_case("stop rule", 80, 128, 7, 200, rel_tol=1e-3)
    ok &= solve_case("multi-block pass (V=1)", 300, 64, 13, 3, env={"PDZ_STREAM_K": "1"})
    ok &= batch_case()
    ok &= slab_case()
    print("ALL OK" if ok else "FAILED", flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
