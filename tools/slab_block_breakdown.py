"""Where one slab block's device time goes (pdz_fixed_point_sweeps_from, config
4 geometry, k sweeps): per-kernel durations from torch.profiler.
usage: python tools/slab_block_breakdown.py [rows] [k]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2506_08793_b200 as pdz  # noqa: E402
from paper_2506_08793_b200 import _native as nat  # noqa: E402
from paper_2506_08793_b200.solver import _params  # noqa: E402

TAU = 0.9 * 2.0 / (8.0 / 1e-3 + 0.5)
E = int(sys.argv[1]) if len(sys.argv) > 1 else 1128
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
W, K = 3840, 25
lib = nat.lib()
dev = nat.device()
cfg = pdz.SolverConfig(tau=TAU, sigma=4.0, kernel_size=K, max_iters=500, rel_tol=1e-300)
rng = np.random.default_rng(0)
u = torch.from_numpy(rng.uniform(0, 1, (3, E, W)).astype(np.float32)).to(dev)
phi = torch.from_numpy(rng.uniform(-0.2, 1.2, (3, E, W)).astype(np.float32)).to(dev)
lam = torch.from_numpy(rng.uniform(0.02, 0.5, (E, W)).astype(np.float32)).to(dev)
prm = _params(E, W, 3, 3, cfg, tau=TAU, max_iters=k)
ws = torch.empty(lib.pdz_solve_workspace_bytes(prm), dtype=torch.uint8, device=dev)
out = torch.empty_like(u)
sums = torch.empty((k, 3), dtype=torch.float64, device=dev)
failed = torch.empty(3, dtype=torch.int32, device=dev)


def run():
    nat.check(lib.pdz_fixed_point_sweeps_from(
        prm, nat.ptr(u), nat.ptr(phi), nat.ptr(lam), 48, E - 48, nat.ptr(out),
        nat.ptr(sums), nat.ptr(failed), nat.ptr(ws), ws.numel(), nat.stream_ptr()))


for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    run()
e1.record()
e1.synchronize()
print(f"rows {E} k {k}: {e0.elapsed_time(e1) / 10:.4f} ms per block (10 back to back)")
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        run()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12, max_name_column_width=60))
