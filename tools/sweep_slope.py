"""Time the streaming solve for several iteration counts: slope = per-sweep
cost, intercept = fixed launch/setup cost.  usage: sweep_slope.py [size] [k]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_08793_b200 as pdz  # noqa: E402
from paper_2506_08793_b200 import _native as nat  # noqa: E402
from paper_2506_08793_b200.solver import (_front_end, _image_dev, _lambda_mode,  # noqa: E402
                                          _params, prepare_problem)
from paper_2506_08793_b200.synthetic import make_hazy_scene  # noqa: E402

size = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
k = int(sys.argv[2]) if len(sys.argv) > 2 else 19
tau = 0.9 * 2.0 / (8.0 / 1e-3 + 0.5)
lib = nat.lib()
img_dev, is_f64 = _image_dev(torch.from_numpy(make_hazy_scene(size, size, 2, 0).hazy))
flags = frozenset(("no-multiscale", "no-guided"))
res = []
for iters in (25, 50, 100, 200, 400):
    cfg = pdz.SolverConfig(tau=tau, sigma=k / 6.0, kernel_size=k, max_iters=iters, rel_tol=1e-300)
    t_dev, a_dev = _front_end(img_dev, is_f64, cfg, flags)
    phi, lam = prepare_problem(img_dev, is_f64, t_dev, a_dev, cfg, _lambda_mode(flags, cfg))
    prm = _params(size, size, 3, 3, cfg)
    ws = torch.empty(lib.pdz_solve_workspace_bytes(prm), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        nat.check(lib.pdz_fixed_point_sweeps_async(prm, nat.ptr(phi), nat.ptr(lam), nat.ptr(ws),
                                                   ws.numel(), nat.stream_ptr()))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        nat.check(lib.pdz_fixed_point_sweeps_async(prm, nat.ptr(phi), nat.ptr(lam), nat.ptr(ws),
                                                   ws.numel(), nat.stream_ptr()))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    res.append((iters, ms))
    print(f"iters {iters:4d}: {ms*1e3:9.1f} us  ({ms*1e3/iters:6.2f} us/sweep)  kind "
          f"{lib.pdz_sweep_kernel_kind(prm)}", flush=True)
(i0, t0), (i1, t1) = res[1], res[-1]
print(f"slope {1e3*(t1-t0)/(i1-i0):.2f} us/sweep, intercept {1e3*(t0 - (t1-t0)/(i1-i0)*i0):.1f} us")
