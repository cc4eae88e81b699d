"""Per-CTA wait profile of the streaming solve (PDZ_PROF=1 debug build hook).
usage: PDZ_PROF=1 prof_stream.py [size] [k] [iters]"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_08793_b200 as pdz  # noqa: E402
from paper_2506_08793_b200 import _native as nat  # noqa: E402
from paper_2506_08793_b200.solver import (_front_end, _image_dev, _lambda_mode,  # noqa: E402
                                          _params, prepare_problem)
from paper_2506_08793_b200.synthetic import make_hazy_scene  # noqa: E402

size = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
k = int(sys.argv[2]) if len(sys.argv) > 2 else 19
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 200
chans = int(os.environ.get("PROF_C", "3"))
tau = 0.9 * 2.0 / (8.0 / 1e-3 + 0.5)
lib = nat.lib()
img = make_hazy_scene(size, size, 2, 0).hazy
if chans == 1:
    img = np.ascontiguousarray(img[:, :, :1])
img_dev, is_f64 = _image_dev(torch.from_numpy(img))
flags = frozenset(("no-multiscale", "no-guided"))
cfg = pdz.SolverConfig(tau=tau, sigma=k / 6.0, kernel_size=k, max_iters=iters, rel_tol=1e-300)
t_dev, a_dev = _front_end(img_dev, is_f64, cfg, flags)
phi, lam = prepare_problem(img_dev, is_f64, t_dev, a_dev, cfg, _lambda_mode(flags, cfg))
prm = _params(size, size, chans, chans, cfg)
ws = torch.empty(lib.pdz_solve_workspace_bytes(prm), dtype=torch.uint8, device="cuda")
for _ in range(3):
    nat.check(lib.pdz_fixed_point_sweeps_async(prm, nat.ptr(phi), nat.ptr(lam), nat.ptr(ws),
                                               ws.numel(), nat.stream_ptr()))
torch.cuda.synchronize()
buf = np.zeros((8192, 16), dtype=np.int64)
lib.pdz_debug_prof.argtypes = [ctypes.c_void_p, ctypes.c_int]
lib.pdz_debug_prof(buf.ctypes.data, 8192)
G = int(((buf[:4096, 6] > 0) & (buf[:4096, 12] > 0)).sum())
g = buf[:G]
sv = buf[G + 1:2 * G + 1]
names = ["total", "grant", "topbar", "mbar", "hbar", "flushbar", "blocks", "defers",
         "mirror", "hpass", "vpass", "prefetch", "next", "compute", "towait"]
os.makedirs("gpurun_out", exist_ok=True)
np.save("gpurun_out/prof_raw.npy", buf[:2 * G + 1])
print(f"G={len(g)}  iters={iters}  per-sweep us (mean / min / max over CTAs):")
for i, n in enumerate(names):
    v = g[:, i] / iters if i in (6, 7) else g[:, i] / (1e3 * iters)
    print(f"  {n:9s} {v.mean():8.3f} {v.min():8.3f} {v.max():8.3f}")
snames = ["fence_ns", "fences", "post2issue", "issues", "grantlat", "waitwr_ns", "depfail", "store_ns"]
print("service warp per sweep (mean / min / max):")
for i, n in enumerate(snames):
    v = sv[:, i] / iters
    if i in (0, 2, 4, 5, 7):
        v = v / 1e3
    if i == 2:
        v = sv[:, 2] / np.maximum(sv[:, 3], 1) / 1e3  # per issue
    print(f"  {n:9s} {v.mean():8.3f} {v.min():8.3f} {v.max():8.3f}")
print("  fence us each", (sv[:, 0].sum() / max(1, sv[:, 1].sum())) / 1e3)
S = ((size + 63) // 64) * size
order = np.argsort(g[:, 1])
print("slowest CTAs (least grant wait): cta strip y0 y1 grant_us/sweep")
for i in order[:12]:
    L0, L1 = i * S // G, (i + 1) * S // G
    print(f"  {i:4d} strip {L0 // size:2d} rows {L0 % size:4d}-{(L1 - 1) % size:4d}  " +
          " ".join(f"{n}={g[i, j] / 1e3 / iters:6.2f}" for j, n in enumerate(names)
                   if j not in (0, 6, 7)))
print("fastest:")
for i in order[-5:]:
    L0, L1 = i * S // G, (i + 1) * S // G
    print(f"  {i:4d} strip {L0 // size:2d} rows {L0 % size:4d}-{(L1 - 1) % size:4d}  " +
          " ".join(f"{n}={g[i, j] / 1e3 / iters:6.2f}" for j, n in enumerate(names)
                   if j not in (0, 6, 7)))
print("slowest CTAs by vpass:")
for i in np.argsort(-g[:, 10])[:16]:
    L0, L1 = i * S // G, (i + 1) * S // G
    print(f"  {i:4d} strip {L0 // size:2d} rows {L0 % size:4d}-{(L1 - 1) % size:4d}  "
          f"vpass={g[i, 10] / 1e3 / iters:6.2f} hpass={g[i, 9] / 1e3 / iters:6.2f} "
          f"mbar={g[i, 3] / 1e3 / iters:6.2f}")
print("fastest by vpass:", ", ".join(f"{i}:{g[i, 10] / 1e3 / iters:.2f}" for i in np.argsort(g[:, 10])[:6]))

print("per-CTA compute (data ready -> end barrier) and lead-warp wait (loop top -> data), us/sweep:")
comp = g[:, 13] / 1e3 / iters
wt = g[:, 14] / 1e3 / iters
for i in np.argsort(-comp)[:20]:
    print(f"  cta {i:4d} compute {comp[i]:6.2f}  wait {wt[i]:6.2f}  hpass {g[i, 9] / 1e3 / iters:5.2f} vpass {g[i, 10] / 1e3 / iters:5.2f}")
print("compute: mean %.2f min %.2f max %.2f" % (comp.mean(), comp.min(), comp.max()))
