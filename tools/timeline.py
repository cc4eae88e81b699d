"""Dependency timeline of the persistent solve (PDZ_PROFILE build + PDZ_PROF=1):
for every (CTA, pass) -- when its IN tile was wanted (generated, buffer free),
when the neighbours it depends on had published the previous pass of the
channel, when the service warp issued the load, and when the compute warps
started / stopped waiting for it.  Config-2 geometry (per-strip partition).
usage: PDZ_LIB_NAME=libpdz_prof.so PDZ_PROF=1 python tools/timeline.py"""
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

size, k, iters, C = 1024, 19, 200, 3
R = k // 2
tau = 0.9 * 2.0 / (8.0 / 1e-3 + 0.5)
lib = nat.lib()
img = make_hazy_scene(size, size, 2, 0).hazy
img_dev, is_f64 = _image_dev(torch.from_numpy(img))
flags = frozenset(("no-multiscale", "no-guided"))
cfg = pdz.SolverConfig(tau=tau, sigma=k / 6.0, kernel_size=k, max_iters=iters, rel_tol=1e-300)
t_dev, a_dev = _front_end(img_dev, is_f64, cfg, flags)
phi, lam = prepare_problem(img_dev, is_f64, t_dev, a_dev, cfg, _lambda_mode(flags, cfg))
prm = _params(size, size, C, C, cfg)
ws = torch.empty(lib.pdz_solve_workspace_bytes(prm), dtype=torch.uint8, device="cuda")
for _ in range(2):
    nat.check(lib.pdz_fixed_point_sweeps_async(prm, nat.ptr(phi), nat.ptr(lam), nat.ptr(ws),
                                               ws.numel(), nat.stream_ptr()))
torch.cuda.synchronize()
buf = np.zeros((262144, 16), dtype=np.int64)
lib.pdz_debug_prof.argtypes = [ctypes.c_void_p, ctypes.c_int]
lib.pdz_debug_prof(buf.ctypes.data, 262144)
tl = buf.reshape(-1)[131072:131072 + 5 * 256 * 2048].reshape(5, 256, 2048).astype(np.float64)
pub, iss, want, ws0, ws1 = tl
G = int((iss[:, 10] > 0).sum())
# per-strip partition of config 2 (pdz_solver.cuh part_start): 16 strips, k = 9, bonus 1
nstr, kps, bonus = size // 64, 9, 1
def part_start(i):
    r = i
    if r < kps + bonus:
        s, t, ks = 0, r, kps + bonus
    else:
        r -= kps + bonus
        s = 1 + r // kps
        if s >= nstr - 1:
            s, t, ks = nstr - 1, r - (nstr - 2) * kps, kps + bonus
        else:
            t, ks = r - (s - 1) * kps, kps
    return s * size + (t * size) // ks
starts = [part_start(i) for i in range(G)] + [nstr * size]
def cta_of(L):
    return int(np.searchsorted(starts, L, side="right") - 1)
deps = []
for i in range(G):
    L0, L1 = starts[i], starts[i + 1]
    s, y0, y1 = L0 // size, L0 % size, (L1 - 1) % size + 1
    d = set()
    for s2 in (s - 1, s, s + 1):
        if 0 <= s2 < nstr:
            for y in (max(0, y0 - R), min(size - 1, y1 - 1 + R)):
                pass
            lo, hi = cta_of(s2 * size + max(0, y0 - R)), cta_of(s2 * size + min(size, y1 + R) - 1)
            d.update(range(lo, hi + 1))
    deps.append(sorted(d))
rows = []
for i in range(G):
    for kk in range(C + 1, iters * C + 1):
        dr = max(pub[d, kk - C] for d in deps[i])
        rows.append((i, kk, want[i, kk], dr, iss[i, kk], ws0[i, kk], ws1[i, kk]))
a = np.array(rows)
w, dr, isu, s0, s1 = a[:, 2], a[:, 3], a[:, 4], a[:, 5], a[:, 6]
ready = np.maximum(w, dr)
print(f"G={G}, {len(a)} (cta, pass) samples, ns")
print(f"  IN wait (compute warps)           mean {np.mean(s1 - s0):7.0f}  p50 {np.median(s1 - s0):7.0f}  p90 {np.percentile(s1 - s0, 90):7.0f}")
print(f"  deps later than buffer-free       frac {np.mean(dr > w):.2f}  mean excess {np.mean(np.maximum(0, dr - w)):7.0f}")
print(f"  issue - max(want, deps) (service) mean {np.mean(isu - ready):7.0f}  p50 {np.median(isu - ready):7.0f}  p90 {np.percentile(isu - ready, 90):7.0f}")
print(f"  wait end - issue (TMA, if waited) mean {np.mean((s1 - isu)[s1 - s0 > 300]):7.0f}")
print(f"  wait start - issue                mean {np.mean(s0 - isu):7.0f}  (negative: issued after the warps wanted it)")
late = s1 - s0 > 300
print(f"  blocks that waited > 300 ns: {np.mean(late):.2f};  of those deps-bound {np.mean((dr > w)[late]):.2f}")
print(f"  for waited blocks: want->wstart {np.mean((s0 - w)[late]):7.0f}  deps->wstart {np.mean((s0 - dr)[late]):7.0f}  svc lat {np.mean((isu - ready)[late]):7.0f}  tma {np.mean((s1 - isu)[late]):7.0f}")
# publication latency: our own publication of pass kk vs our compute end (next block's wait start ~ block end)
pubk = np.array([[pub[i, kk] for kk in range(C + 1, iters * C)] for i in range(G)])
endk = np.array([[ws0[i, kk + 1] for kk in range(C + 1, iters * C)] for i in range(G)])
print(f"  publication - next IN wait start (~block end) mean {np.mean(pubk - endk):7.0f}")
