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
    stop = os.environ.get("STOPRULE") == "1"  # fixed_point_solve path: stop rule armed
    import numpy as np
    out = torch.empty_like(phi)
    hn = np.zeros((iters, 3)); hi = np.zeros(3, np.int32)
    hc = np.zeros(3, np.int32); hf = np.zeros(3, np.int32)

    def run():
        if stop:
            nat.check(lib.pdz_fixed_point_solve(prm, nat.ptr(phi), nat.ptr(lam), nat.ptr(out),
                                                hn.ctypes.data, hi.ctypes.data, hc.ctypes.data,
                                                hf.ctypes.data, nat.ptr(ws), ws.numel(),
                                                nat.stream_ptr()))
        else:
            nat.check(lib.pdz_fixed_point_sweeps_async(prm, nat.ptr(phi), nat.ptr(lam),
                                                       nat.ptr(ws), ws.numel(), nat.stream_ptr()))

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    lib.pdz_time_sweep_kernels(1)
    ms = 0.0
    for _ in range(5):
        run()
        torch.cuda.synchronize()
        ms += lib.pdz_last_sweep_kernel_ms() / 5
    lib.pdz_time_sweep_kernels(0)
    res.append((iters, ms))
    print(f"iters {iters:4d}: {ms*1e3:9.1f} us  ({ms*1e3/iters:6.2f} us/sweep)  kind "
          f"{lib.pdz_sweep_kernel_kind(prm)}", flush=True)
(i0, t0), (i1, t1) = res[1], res[-1]
print(f"slope {1e3*(t1-t0)/(i1-i0):.2f} us/sweep, intercept {1e3*(t0 - (t1-t0)/(i1-i0)*i0):.1f} us")
