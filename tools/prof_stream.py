"""Per-CTA time profile of the persistent solve (PDZ_PROFILE build + PDZ_PROF=1).
usage: PDZ_LIB_NAME=libpdz_prof.so PDZ_PROF=1 python tools/prof_stream.py [size] [k] [iters]"""
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
if os.environ.get("PDZ_NOSTOP"):  # experiment: fixed iterations without the stop-rule machinery
    prm.rel_tol = -1.0
ws = torch.empty(lib.pdz_solve_workspace_bytes(prm), dtype=torch.uint8, device="cuda")
for _ in range(3):
    nat.check(lib.pdz_fixed_point_sweeps_async(prm, nat.ptr(phi), nat.ptr(lam), nat.ptr(ws),
                                               ws.numel(), nat.stream_ptr()))
torch.cuda.synchronize()
buf = np.zeros((8192, 16), dtype=np.int64)
lib.pdz_debug_prof.argtypes = [ctypes.c_void_p, ctypes.c_int]
lib.pdz_debug_prof(buf.ctypes.data, 8192)
G = int((buf[0:4096:2, 7] > 0).sum())
w0 = buf[0:2 * G:2]
wl = buf[1:2 * G:2]
sv = buf[2 * G + 2:3 * G + 2]
pv = buf[3 * G + 4:4 * G + 4]
os.makedirs("gpurun_out", exist_ok=True)
np.save("gpurun_out/prof_raw.npy", buf[:4 * G + 4])
names = ["total", "in_wait", "hpass", "hbar", "pl_wait", "vpass", "report+bar", "blocks"]
per = lambda x: x / iters  # cycles per sweep
print(f"G={G} iters={iters}  cycles per sweep (mean / min / max over CTAs)")
for lab, arr in (("warp 0", w0), (f"warp last", wl)):
    print(lab)
    for i, n in enumerate(names):
        v = per(arr[:, i].astype(float))
        print(f"  {n:11s} {v.mean():9.1f} {v.min():9.1f} {v.max():9.1f}")
sn = ["rounds", "scan_cyc", "publish", "sleeps", "done_ev", "iss2done"]
print("service warp per sweep:")
for i, n in enumerate(sn):
    v = sv[:, i].astype(float) / iters
    if i == 5:
        v = sv[:, 5] / np.maximum(sv[:, 4], 1)
    print(f"  {n:9s} {v.mean():9.1f} {v.min():9.1f} {v.max():9.1f}")
busy = (w0[:, 2] + w0[:, 5]) / iters
print("warp0 busy (h+v) per sweep: mean %.0f max %.0f (cta %d)" % (busy.mean(), busy.max(), busy.argmax()))
for i in np.argsort(-(w0[:, 1] + w0[:, 4]))[:8]:
    print(f"  most waiting cta {i}: in_wait {w0[i,1]/iters:.0f} pl_wait {w0[i,4]/iters:.0f} hbar {w0[i,3]/iters:.0f}")
for i in np.argsort(w0[:, 1] + w0[:, 4])[:8]:
    print(f"  least waiting cta {i}: in_wait {w0[i,1]/iters:.0f} pl_wait {w0[i,4]/iters:.0f} hbar {w0[i,3]/iters:.0f} vpass {w0[i,5]/iters:.0f}")

n8, s9, n10, s11 = (w0[:, 8].sum(), w0[:, 9].sum(), w0[:, 10].sum(), w0[:, 11].sum())
print(f"warp0 waits: {n8/G/iters:.2f}/sweep found the load unissued (avg issue {s9/max(n8,1):.0f} cyc after wait start); "
      f"{n10/G/iters:.2f}/sweep waited on an issued load (avg ready {s11/max(n10,1):.0f} cyc after issue)")

rp = sv[:, 8:16].astype(float) / iters
print("service round cycles per sweep: done-test %.0f  gen %.0f  scan %.0f  grant+tma %.0f  sleep %.0f  rest %.0f  reduce %.0f  release-store %.0f" % tuple(rp.mean(axis=0)))
