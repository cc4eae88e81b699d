import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_2506_08793_b200 as pdz
from paper_2506_08793_b200 import synthetic as SYN
from conftest import TAU_STABLE
FLAGS = ("no-multiscale", "no-guided")
c = SYN.BENCH_CONFIGS[3]
cfg = pdz.SolverConfig(tau=TAU_STABLE, sigma=c["sigma"], kernel_size=c["kernel_size"], patch_radius=c["patch_radius"], max_iters=90, rel_tol=3e-3)
imgs = [SYN.make_hazy_scene(480, 640, 3, i).hazy.astype(np.float64) for i in range(16)]
outs = []
for rep in range(3):
    out, res = pdz.dehaze_batch(imgs, cfg, ablation=FLAGS)
    outs.append(out)
    if rep: print("batch rep", rep, "equal to rep0:", np.array_equal(out, outs[0]))
out = outs[0]
for i in range(16):
    o, r = pdz.dehaze(imgs[i], cfg, ablation=FLAGS)
    o2, r2 = pdz.dehaze(imgs[i], cfg, ablation=FLAGS)
    its = [t.iterations_run for t in res[i].traces]; its1 = [t.iterations_run for t in r.traces]
    neq = [x.residual_norms == y.residual_norms for x, y in zip(res[i].traces, r.traces)]
    d = out[i] != o
    msg = f"img {i} its batch {its} single {its1} norms_eq {neq} single_repeat_eq {np.array_equal(o,o2)} mism {int(d.sum())}"
    for ch in range(3):
        ys, xs = np.nonzero(d[:, :, ch])
        if len(ys): msg += f" | ch{ch}: n={len(ys)} rows {ys.min()}-{ys.max()} cols {xs.min()}-{xs.max()}"
    print(msg)
