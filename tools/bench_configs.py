"""Device-resident solve throughput for every BASELINE config on one GPU (the
bench.py line is config 2 only).  Seeded synthetic inputs; the
solve runs a bounded number of sweeps (sampled, labelled) and the per-sweep
device time of the persistent launch is reported with its HBM-roofline
fraction (40 B per RGB pixel per sweep).
usage: python tools/bench_configs.py [--iters N]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2506_08793_b200 as pdz  # noqa: E402
from paper_2506_08793_b200 import _native as nat  # noqa: E402
from paper_2506_08793_b200.solver import (_front_end, _image_dev, _lambda_mode,  # noqa: E402
                                          _params, prepare_problem)
from paper_2506_08793_b200.synthetic import make_hazy_scene  # noqa: E402

TAU = 0.9 * 2.0 / (8.0 / 1e-3 + 0.5)
CONFIGS = [  # name, H, W, images, K, sigma, patch radius, iterations of the config
    ("config1 256x256 K=13", 256, 256, 1, 13, 2.0, 7, 50),
    ("config2 1024x1024 K=19", 1024, 1024, 1, 19, 3.0, 7, 200),
    ("config3 640x480 x256 K=13", 480, 640, 256, 13, 2.0, 7, 100),
    ("config4 3840x2160 K=25", 2160, 3840, 1, 25, 4.0, 15, 500),
    ("config5 7680x4320 K=49", 4320, 7680, 1, 49, 8.0, 7, 2000),
]


def peak():
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(__file__)),
                               "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6650.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=40)
    ap.add_argument("--only", default="", help="comma-separated config numbers (1-5)")
    args = ap.parse_args()
    lib = nat.lib()
    flags = frozenset(("no-multiscale", "no-guided"))
    pk = peak()
    only = {int(x) for x in args.only.split(",") if x}
    for ci, (name, h, w, nimg, k, sigma, pr, full_iters) in enumerate(CONFIGS, 1):
        if only and ci not in only:
            continue
        iters = min(args.iters, full_iters)
        cfg = pdz.SolverConfig(tau=TAU, sigma=sigma, kernel_size=k, patch_radius=pr,
                               max_iters=iters, rel_tol=1e-300)
        phi = torch.empty((nimg * 3, h, w), dtype=torch.float32, device="cuda")
        lam = torch.empty((nimg, h, w), dtype=torch.float32, device="cuda")
        distinct = min(nimg, 8)  # front end of 8 distinct images, tiled over the batch
        for i in range(distinct):
            img = make_hazy_scene(h, w, 3, i).hazy
            img_dev, is_f64 = _image_dev(torch.from_numpy(img))
            t_dev, a_dev = _front_end(img_dev, is_f64, cfg, flags)
            prepare_problem(img_dev, is_f64, t_dev, a_dev, cfg, _lambda_mode(flags, cfg),
                            phi=phi[3 * i:3 * i + 3], lam=lam[i])
        for i in range(distinct, nimg):
            phi[3 * i:3 * i + 3].copy_(phi[3 * (i % distinct):3 * (i % distinct) + 3])
            lam[i].copy_(lam[i % distinct])
        prm = _params(h, w, 3 * nimg, 3, cfg)
        ws = torch.empty(lib.pdz_solve_workspace_bytes(prm), dtype=torch.uint8, device="cuda")

        def run():
            nat.check(lib.pdz_fixed_point_sweeps_async(prm, nat.ptr(phi), nat.ptr(lam),
                                                       nat.ptr(ws), ws.numel(),
                                                       nat.stream_ptr()))

        run()
        torch.cuda.synchronize()
        lib.pdz_time_sweep_kernels(1)
        reps = 3
        ms = 0.0
        for _ in range(reps):
            run()
            torch.cuda.synchronize()
            ms += lib.pdz_last_sweep_kernel_ms() / reps
        lib.pdz_time_sweep_kernels(0)
        px = h * w * nimg
        mpix = px * iters / (ms / 1e3) / 1e6
        gbs = 40.0 * px * iters / (ms / 1e3) / 1e9
        print(json.dumps({"config": name, "sweeps_timed": iters, "full_iterations": full_iters,
                          "kernel": int(lib.pdz_sweep_kernel_kind(prm)),
                          "us_per_sweep": round(ms * 1e3 / iters, 2),
                          "mpix_it_per_s": round(mpix), "hbm_frac": round(gbs / pk, 3)}),
              flush=True)
        del phi, lam, ws
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
