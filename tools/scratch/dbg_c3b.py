import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_2506_08793_b200 as pdz
from paper_2506_08793_b200 import synthetic as SYN, _native as nat
from paper_2506_08793_b200.solver import _params
from conftest import TAU_STABLE
FLAGS = ("no-multiscale", "no-guided")
c = SYN.BENCH_CONFIGS[3]
imgs = [SYN.make_hazy_scene(480, 640, 3, i).hazy.astype(np.float64) for i in range(16)]
for iters in (1, 2, 3, 4, 8):
    cfg = pdz.SolverConfig(tau=TAU_STABLE, sigma=c["sigma"], kernel_size=c["kernel_size"], patch_radius=c["patch_radius"], max_iters=iters, rel_tol=1e-300)
    if iters == 1:
        print("plan batch", nat.plan_info(_params(480, 640, 48, 3, cfg)))
        print("plan single", nat.plan_info(_params(480, 640, 3, 3, cfg)))
    out, res = pdz.dehaze_batch(imgs, cfg, ablation=FLAGS)
    for i in (0, 7):
        o, r = pdz.dehaze(imgs[i], cfg, ablation=FLAGS)
        d = out[i] != o
        msg = f"iters {iters} img {i} mism {int(d.sum())} maxabs {np.abs(out[i]-o).max():.3g}"
        for ch in range(3):
            ys, xs = np.nonzero(d[:, :, ch])
            if len(ys): msg += f" | ch{ch}: n={len(ys)} rows {ys.min()}-{ys.max()} cols {xs.min()}-{xs.max()} first {list(zip(ys[:6], xs[:6]))}"
        print(msg)
