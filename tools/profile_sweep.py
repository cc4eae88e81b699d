"""Profiling driver: the config-2 solve (1024^2 x 3, K=19) for a few sweeps.

    python tools/profile_sweep.py [--iters N] [--k K] [--size S]
Used under ncu (launch list / --set full) -- never for bench numbers.
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2506_08793_b200 as pdz  # noqa: E402
from paper_2506_08793_b200 import _native as nat  # noqa: E402
from paper_2506_08793_b200.solver import (DeviceProblem, _front_end, _image_dev,  # noqa: E402
                                          _lambda_mode, _params, prepare_problem)
from paper_2506_08793_b200.synthetic import make_hazy_scene  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--k", type=int, default=19)
ap.add_argument("--sigma", type=float, default=3.0)
ap.add_argument("--size", type=int, default=1024)
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()

tau = 0.9 * 2.0 / (8.0 / 1e-3 + 0.5)
cfg = pdz.SolverConfig(tau=tau, sigma=args.sigma, kernel_size=args.k, max_iters=args.iters,
                       rel_tol=1e-300)
img = torch.from_numpy(make_hazy_scene(args.size, args.size, 2, 0).hazy)
img_dev, is_f64 = _image_dev(img)
flags = frozenset(("no-multiscale", "no-guided"))
t_dev, a_dev = _front_end(img_dev, is_f64, cfg, flags)
phi, lam = prepare_problem(img_dev, is_f64, t_dev, a_dev, cfg, _lambda_mode(flags, cfg))
prm = _params(args.size, args.size, 3, 3, cfg)
lib = nat.lib()
ws = torch.empty(lib.pdz_solve_workspace_bytes(prm), dtype=torch.uint8, device="cuda")
for _ in range(args.reps):
    nat.check(lib.pdz_fixed_point_sweeps_async(prm, nat.ptr(phi), nat.ptr(lam), nat.ptr(ws),
                                               ws.numel(), nat.stream_ptr()))
torch.cuda.synchronize()
print("ok")
