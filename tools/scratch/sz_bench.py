"""usage: sz_bench.py H W K sigma [iters]  -- device-resident solve time for one custom size."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2506_08793_b200 as pdz
from paper_2506_08793_b200 import _native as nat
from paper_2506_08793_b200.solver import _front_end, _image_dev, _lambda_mode, _params, prepare_problem
from paper_2506_08793_b200.synthetic import make_hazy_scene
h, w, k, sigma = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 200
TAU = 0.9 * 2.0 / (8.0 / 1e-3 + 0.5)
lib = nat.lib()
flags = frozenset(("no-multiscale", "no-guided"))
cfg = pdz.SolverConfig(tau=TAU, sigma=sigma, kernel_size=k, patch_radius=7, max_iters=iters, rel_tol=1e-300)
img = make_hazy_scene(h, w, 3, 0).hazy
img_dev, is_f64 = _image_dev(torch.from_numpy(img))
t_dev, a_dev = _front_end(img_dev, is_f64, cfg, flags)
phi, lam = prepare_problem(img_dev, is_f64, t_dev, a_dev, cfg, _lambda_mode(flags, cfg))
prm = _params(h, w, 3, 3, cfg)
ws = torch.empty(lib.pdz_solve_workspace_bytes(prm), dtype=torch.uint8, device="cuda")
def run():
    nat.check(lib.pdz_fixed_point_sweeps_async(prm, nat.ptr(phi), nat.ptr(lam), nat.ptr(ws), ws.numel(), nat.stream_ptr()))
run(); torch.cuda.synchronize()
lib.pdz_time_sweep_kernels(1)
ms = []
for _ in range(5):
    run(); torch.cuda.synchronize(); ms.append(lib.pdz_last_sweep_kernel_ms())
m = sorted(ms)[2]
print(json.dumps({"lib": os.environ.get("PDZ_LIB_NAME", "libpdz.so"), "hw": [h, w], "plan": nat.plan_info(prm), "us_per_sweep": round(m * 1e3 / iters, 3), "mpix_it_s": round(h * w * iters / m / 1e3)}))
