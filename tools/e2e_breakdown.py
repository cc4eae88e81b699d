"""Where the e2e time of one config-2 dehaze() goes (torch.profiler, CUDA
activity): kernel / memcpy totals and the host-side gaps."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_08793_b200 as pdz  # noqa: E402
from paper_2506_08793_b200.synthetic import make_hazy_scene  # noqa: E402

TAU = 0.9 * 2.0 / (8.0 / 1e-3 + 0.5)
cfg = pdz.SolverConfig(tau=TAU, sigma=3.0, kernel_size=19, patch_radius=7, max_iters=200,
                       rel_tol=1e-300)
host = torch.from_numpy(make_hazy_scene(1024, 1024, 2, 0).hazy).pin_memory()
def step():
    out, _ = pdz.dehaze(host, cfg, ablation=("no-multiscale", "no-guided"))
    return out


for _ in range(3):
    step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    step()
torch.cuda.synchronize()
print(f"wall per step {(time.perf_counter() - t0) / 5 * 1e3:.3f} ms")
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30))
