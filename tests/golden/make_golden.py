"""Generate the golden fixtures in tests/golden/ by running the REAL reference.

Run in the build container, where the reference tree is mounted read-only:

    python tests/golden/make_golden.py            # writes tests/golden/*.npz

The reference package is imported from /root/reference/pkg/src (pure
Python, numpy + scipy); nothing is copied from it.  The GPU box never needs
this script: the .npz files it writes are committed and travel with the repo.

Fixtures
  operators.npz    divergence_term / gaussian_convolve / tau_stability_bound /
                   adaptive_lambda / diffusion_coefficient on seeded fields
  frontend.npz     dark_channel, multiscale_dark_channel, airlight (value and
                   the stable-argsort selection order), transmission,
                   reconstruct, box_mean / guided_filter / refine_transmission
  solve.npz        fixed_point_step, fixed_point_solve (fixed iterations, stop
                   rule, no-edge, given lambda), short dehaze runs
  golden_trace.npz the reference demo's residual trace (demos/solver_convergence.py),
                   checked here against demos/out/residual_traces.csv
  config1.npz      BASELINE config 1 (256x256x3, patch 15, sigma 2 / K 13,
                   50 iterations, tau = TAU_STABLE) through dehaze
  cli.npz          the reference command line (synthesize / dehaze / evaluate)
                   on small Netpbm files: input and output bytes
"""

from __future__ import annotations

import csv
import hashlib
import math
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_DEMOS = "/root/reference/pkg/demos"
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REPO)

import pdehaze as ref  # noqa: E402

from paper_2506_08793_b200.synthetic import make_hazy_scene  # noqa: E402

TAU_STABLE = 0.9 * 2.0 / (8.0 / 1e-3 + 0.5)
ABL = ("no-multiscale", "no-guided")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def selection(dark, fraction):
    """The indices the reference's estimate_atmospheric_light averages
    (scattering.py:102-105), recomputed with the reference's own expression."""
    count = math.ceil(fraction * dark.size)
    return np.argsort(-dark.ravel(), kind="stable")[:count]


def tie_image(rng, h, w):
    """Coarsely quantised image: many exactly equal dark values (tie-break test)."""
    return np.round(rng.random((h, w, 3)) * 8) / 8


def operators():
    rng = np.random.default_rng(20260101)
    out = {}
    shapes = [(2, 2), (2, 5), (3, 3), (6, 6), (7, 9), (16, 13), (33, 40)]
    for i, s in enumerate(shapes):
        u = rng.standard_normal(s) * (10.0 ** rng.integers(-2, 2))
        out[f"div_u_{i}"] = u
        out[f"div_edge_{i}"] = ref.divergence_term(u, 1e-3)
        out[f"div_lap_{i}"] = ref.divergence_term(u, 1e-3, edge_preserving=False)
        lam = rng.random(s) * 0.6
        out[f"tau_lam_{i}"] = lam
        out[f"tau_{i}"] = np.array(ref.tau_stability_bound(u, lam, 1e-3))
    gauss_cases = [((4, 4), 2.0, 13), ((10, 10), 2.0, 5), ((7, 9), 1.5, 3), ((5, 6), 2.0, 1),
                   ((16, 16), 2.0, 13), ((12, 20), 3.0, 19), ((3, 2), 4.0, 25),
                   ((40, 31), 8.0, 49)]
    for i, (s, sigma, k) in enumerate(gauss_cases):
        f = rng.standard_normal(s)
        out[f"g_in_{i}"] = f
        out[f"g_sigma_{i}"] = np.array(sigma)
        out[f"g_k_{i}"] = np.array(k)
        out[f"g_out_{i}"] = ref.gaussian_convolve(f, sigma, k)
        out[f"g_kernel_{i}"] = ref.gaussian_kernel(sigma, k)
    t = rng.random((15, 17))
    t[0, 0], t[0, 1] = 0.0, 1.0
    out["lam_t"] = t
    out["lam_printed"] = ref.adaptive_lambda(t, 0.5, 3.0)
    out["lam_prose"] = ref.adaptive_lambda(t, 0.7, 2.0, monotonicity="prose")
    g = rng.random(100) * 10
    g[:5] = 0.0
    out["dcoef_g"] = g
    out["dcoef"] = ref.diffusion_coefficient(g, 1e-3)
    np.savez_compressed(os.path.join(HERE, "operators.npz"), **out)


def frontend():
    rng = np.random.default_rng(20260102)
    out = {}
    scenes = [make_hazy_scene(48, 64, 91, 0).hazy.astype(np.float64),
              make_hazy_scene(37, 29, 91, 1).hazy.astype(np.float64),
              tie_image(rng, 40, 52),
              rng.random((9, 11, 3)),
              rng.random((23, 31, 1))]
    scenes[2][5:15, 10:30] = 1.0  # a saturated block: ties at the top value
    for i, img in enumerate(scenes):
        c = img.shape[2]
        out[f"img_{i}"] = img
        a_rand = 0.2 + 0.8 * rng.random(c)
        out[f"arand_{i}"] = a_rand
        for r in (0, 1, 2, 7, 15, 40):
            out[f"dark1_{i}_{r}"] = ref.dark_channel(img, np.ones(c), r)
            out[f"darka_{i}_{r}"] = ref.dark_channel(img, a_rand, r)
        out[f"ms_{i}"] = ref.multiscale_dark_channel(img, np.ones(c), (3, 7, 15))
        out[f"msw_{i}"] = ref.multiscale_dark_channel(img, a_rand, (1, 4), (0.3, 0.7))
        dark = ref.dark_channel(img, np.ones(c), 7)
        for j, frac in enumerate((0.001, 0.03, 0.5, 1.0)):
            out[f"air_{i}_{j}"] = ref.estimate_atmospheric_light(img, dark, frac)
            out[f"pick_{i}_{j}"] = selection(dark, frac)
        out[f"air_ms_{i}"] = ref.estimate_atmospheric_light(img, out[f"ms_{i}"], 0.01)
        out[f"pick_ms_{i}"] = selection(out[f"ms_{i}"], 0.01)
        a = ref.estimate_atmospheric_light(img, dark, 0.001)
        dn = ref.dark_channel(img, a, 7)
        t = ref.estimate_transmission(dn, 0.95)
        out[f"t_{i}"] = t
        out[f"recon_{i}"] = ref.reconstruct(img, t, a, 0.1)
        if min(img.shape[:2]) >= 2:
            out[f"refine_{i}"] = ref.refine_transmission(img, t, 30, 1e-3)
            out[f"refine5_{i}"] = ref.refine_transmission(img, t, 5, 1e-2)
    # mean-order stress: many picked pixels with varied values
    big = rng.random((64, 96, 3))
    dk = ref.dark_channel(big, np.ones(3), 0)
    out["air_big_img"] = big
    out["air_big"] = ref.estimate_atmospheric_light(big, dk, 0.37)
    out["pick_big"] = selection(dk, 0.37)
    f = rng.random((19, 27))
    out["box_in"] = f
    for r in (1, 2, 5, 30):
        out[f"box_{r}"] = ref.box_mean(f, r)
    gd, tg = rng.random((21, 18)), rng.random((21, 18))
    out["gf_guide"], out["gf_target"] = gd, tg
    out["gf_out"] = ref.guided_filter(gd, tg, 3, 1e-2)
    np.savez_compressed(os.path.join(HERE, "frontend.npz"), **out)


def solve():
    rng = np.random.default_rng(20260103)
    out = {}
    cfg = ref.SolverConfig()
    u = rng.random((7, 7))
    src = rng.standard_normal((7, 7))
    lam = rng.random((7, 7)) * 0.5
    out["step_u"], out["step_src"], out["step_lam"] = u, src, lam
    un, nrm = ref.fixed_point_step(u, src, lam, cfg)
    out["step_out"], out["step_norm"] = un, np.array(nrm)
    un, nrm = ref.fixed_point_step(u, src, lam, cfg, edge_preserving=False, tau=1e-3)
    out["step_lap_out"], out["step_lap_norm"] = un, np.array(nrm)
    scene = make_hazy_scene(48, 64, 92, 0)
    img = scene.hazy.astype(np.float64)
    out["solve_img"] = img
    dark = ref.dark_channel(img, np.ones(3), 7)
    a = ref.estimate_atmospheric_light(img, dark)
    t = ref.estimate_transmission(ref.dark_channel(img, a, 7))
    out["solve_t"], out["solve_a"] = t, a
    runs = {
        "fixed": dict(cfg=ref.SolverConfig(tau=TAU_STABLE, sigma=2.0, kernel_size=13,
                                           max_iters=30, rel_tol=1e-300)),
        "k5": dict(cfg=ref.SolverConfig(tau=TAU_STABLE, max_iters=40, rel_tol=1e-300)),
        "stop": dict(cfg=ref.SolverConfig(tau=TAU_STABLE, max_iters=400, rel_tol=2e-3)),
        "noedge": dict(cfg=ref.SolverConfig(tau=0.05, max_iters=25, rel_tol=1e-300),
                       edge_preserving=False),
        "lamgiven": dict(cfg=ref.SolverConfig(tau=TAU_STABLE, max_iters=20, rel_tol=1e-300),
                         lambda_map=np.full(t.shape, 0.3)),
        "k1": dict(cfg=ref.SolverConfig(tau=TAU_STABLE, kernel_size=1, max_iters=15,
                                        rel_tol=1e-300)),
    }
    for name, kw in runs.items():
        cfg = kw.pop("cfg")
        uu, tr = ref.fixed_point_solve(img[:, :, 1], t, float(a[1]), cfg, **kw)
        out[f"solve_{name}_u"] = uu
        out[f"solve_{name}_norms"] = np.array(tr.residual_norms)
        out[f"solve_{name}_meta"] = np.array([tr.iterations_run, int(tr.converged),
                                              tr.tau_used, tr.tau_bound])
    for k, flags in enumerate((ABL, (), ("no-multiscale",), ("no-guided", "no-edge"),
                               ("no-guided", "no-nonlocal"), ("no-guided", "no-adaptive"),
                               ("no-pde",))):
        im = make_hazy_scene(40, 56, 93, k).hazy.astype(np.float64)
        cfg = ref.SolverConfig(tau=TAU_STABLE, max_iters=12, rel_tol=1e-300)
        res, info = ref.dehaze(im, cfg, ablation=flags)
        out[f"dh_img_{k}"] = im
        out[f"dh_flags_{k}"] = np.array(",".join(flags))
        out[f"dh_out_{k}"] = res
        out[f"dh_a_{k}"] = info.airlight
        out[f"dh_t_{k}"] = info.transmission
        out[f"dh_norms_{k}"] = np.array([tr.residual_norms for tr in info.traces])
    np.savez_compressed(os.path.join(HERE, "solve.npz"), **out)


def golden_trace():
    sys.path.insert(0, REF_DEMOS)
    from dehaze_synthetic_scene import build_scene  # reference demo helper

    clean = build_scene(seed=5, size=64)
    t = np.full((64, 64), 0.5)
    hazy = ref.synthesize_haze(clean, t, np.full(3, 0.85))
    channel = hazy[:, :, 1]
    lam = ref.adaptive_lambda(t)
    bound = ref.tau_stability_bound(channel, lam, epsilon=1e-3)
    traces = []
    for tau in (0.2, 0.9 * bound):
        cfg = ref.SolverConfig(tau=tau, max_iters=60, rel_tol=1e-15)
        _, tr = ref.fixed_point_solve(channel, t, 0.85, cfg)
        traces.append(tr.residual_norms)
    # pin against the reference's committed CSV
    with open(os.path.join(REF_DEMOS, "out", "residual_traces.csv"), newline="") as fh:
        rows = list(csv.reader(fh))[1:]
    for ch, it, val in rows:
        assert traces[int(ch)][int(it) - 1] == float(val), (ch, it)
    np.savez_compressed(os.path.join(HERE, "golden_trace.npz"), channel=channel,
                        transmission=t, airlight=np.array(0.85), tau=np.array([0.2, 0.9 * bound]),
                        bound=np.array(bound), norms=np.array(traces))


def config1():
    spec = dict(height=256, width=256)
    scene = make_hazy_scene(spec["height"], spec["width"], 1, 0)
    img = scene.hazy.astype(np.float64)
    cfg = ref.SolverConfig(tau=TAU_STABLE, sigma=2.0, kernel_size=13, patch_radius=7,
                           max_iters=50, rel_tol=1e-300)
    out, info = ref.dehaze(img, cfg, ablation=ABL, workers=3)
    dark = ref.dark_channel(img, np.ones(3), 7)
    np.savez_compressed(
        os.path.join(HERE, "config1.npz"), input_sha=np.array(sha(scene.hazy)),
        out=out.astype(np.float32), airlight=info.airlight, transmission=info.transmission,
        picked=selection(dark, cfg.airlight_fraction).astype(np.int64),
        norms=np.array([tr.residual_norms for tr in info.traces]),
        tau_bound=np.array([tr.tau_bound for tr in info.traces]))


def cli():
    """The reference command line (cli.py) end to end on small Netpbm files:
    synthesize / dehaze (stable tau, default pipeline; no-pde; grayscale) /
    evaluate, plus a commented-header P6 through load_image."""
    import contextlib
    import io
    import tempfile

    from pdehaze.cli import main as ref_main
    from pdehaze.image import load_image as ref_load
    from pdehaze.image import save_image as ref_save

    out = {}
    with tempfile.TemporaryDirectory() as d:
        def path(name):
            return os.path.join(d, name)

        def read(name):
            with open(path(name), "rb") as fh:
                return np.frombuffer(fh.read(), dtype=np.uint8).copy()

        scene = make_hazy_scene(48, 64, 3, 0)
        ref_save(scene.clear.astype(np.float64), path("clean.ppm"))
        rng = np.random.default_rng(77)
        ref_save(rng.uniform(0.2, 0.95, size=(48, 64)), path("tmap.pgm"))
        ref_save(scene.clear.astype(np.float64)[:, :, 1], path("gray.pgm"))
        runs = {
            "synth": ["synthesize", path("clean.ppm"), path("hazy.ppm"), "--t", "0.4",
                      "--airlight", "0.8,0.85,0.9"],
            "synth_map": ["synthesize", path("clean.ppm"), path("hazy_map.ppm"), "--t-map",
                          path("tmap.pgm"), "--airlight", "0.9"],
            "dehaze": ["dehaze", path("hazy.ppm"), path("dehazed.ppm"), "--tau", repr(TAU_STABLE),
                       "--max-iters", "30", "--rel-tol", "1e-300", "--trace", path("trace.csv")],
            "nopde": ["dehaze", path("hazy.ppm"), path("nopde.ppm"), "--tau", repr(TAU_STABLE),
                      "--ablate", "no-pde"],
            "gray": ["dehaze", path("gray.pgm"), path("gray_out.pgm"), "--tau", repr(TAU_STABLE),
                     "--max-iters", "20", "--rel-tol", "1e-300", "--ablate", "no-guided"],
        }
        for key in ("synth", "synth_map", "dehaze", "nopde", "gray"):
            assert ref_main(runs[key]) == 0, key
        for name in ("clean.ppm", "tmap.pgm", "gray.pgm", "hazy.ppm", "hazy_map.ppm",
                     "dehazed.ppm", "nopde.ppm", "gray_out.pgm"):
            out["file_" + name.replace(".", "_")] = read(name)
        with open(path("trace.csv")) as fh:
            out["trace_csv"] = np.array(fh.read())
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            assert ref_main(["evaluate", path("clean.ppm"), path("hazy.ppm")]) == 0
        out["evaluate_json"] = np.array(buf.getvalue().strip())
        # commented header, CRLF-free, comment between every field
        payload = rng.integers(0, 256, size=(5, 7, 3), dtype=np.uint8)
        with open(path("commented.ppm"), "wb") as fh:
            fh.write(b"P6 # magic\n# a comment line\n7 # width\n5\n# maxval next\n255\n")
            fh.write(payload.tobytes())
        out["file_commented_ppm"] = read("commented.ppm")
        out["commented_values"] = ref_load(path("commented.ppm"))
    np.savez_compressed(os.path.join(HERE, "cli.npz"), **out)


if __name__ == "__main__":
    cli()
    operators()
    frontend()
    solve()
    golden_trace()
    config1()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
