import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import __graft_entry__
import paper_2506_08793_b200 as pdz
from paper_2506_08793_b200 import synthetic as SYN
from oracle import pdz_oracle as orc
from conftest import TAU_STABLE
__graft_entry__.build_oracle()
FLAGS = ("no-multiscale", "no-guided")
def cfgn(n, **kw):
    c = SYN.BENCH_CONFIGS[n]
    base = dict(tau=TAU_STABLE, sigma=c["sigma"], kernel_size=c["kernel_size"], patch_radius=c["patch_radius"], max_iters=c["max_iters"], rel_tol=c.get("rel_tol", 1e-300))
    base.update(kw); return pdz.SolverConfig(**base)
# (1)
imgs = [SYN.make_hazy_scene(480, 640, 3, i).hazy.astype(np.float64) for i in range(16)]
cfg = cfgn(3, rel_tol=3e-3, max_iters=90)
out, res = pdz.dehaze_batch(imgs, cfg, ablation=FLAGS)
for i in (0, 5):
    o, r = pdz.dehaze(imgs[i], cfg, ablation=FLAGS)
    d = out[i] != o
    print("img", i, "mism", int(d.sum()), "maxabs", np.abs(out[i]-o).max(), [ (x.iterations_run, y.iterations_run, x.residual_norms == y.residual_norms, max(abs(a-b)/b for a,b in zip(x.residual_norms,y.residual_norms))) for x,y in zip(res[i].traces, r.traces)])
# (2)
c5 = SYN.make_hazy_scene(4320, 7680, 5, 0).hazy.astype(np.float64)
crop = np.ascontiguousarray(c5[100:228, 6000:6384])
for kw in (dict(), dict(max_iters=200, rel_tol=1e-300), dict(max_iters=600, rel_tol=1e-300), dict(max_iters=1200, rel_tol=1e-300)):
    cfg = cfgn(5, **kw)
    out, info = pdz.dehaze(crop, cfg, ablation=FLAGS)
    ro, ra, rt, rtr = orc.run_pipeline(crop, orc.SolverSettings.from_config(cfg), FLAGS, native=True)
    e = np.abs(out - ro)
    idx = np.unravel_index(e.argmax(), e.shape)
    print(kw, "err", e.max(), "at", idx, "iters", [t.iterations_run for t in info.traces], [t.iterations_run for t in rtr], "clamped?", out[idx], ro[idx],
          "norm rel", [max(abs(a-b)/b for a,b in zip(x.residual_norms,y.residual_norms)) for x,y in zip(info.traces, rtr)])
    print("   err percentiles", np.percentile(e, [50, 99, 99.9, 99.99]), "rows of top errs", np.unique(np.argwhere(e > 0.5*e.max())[:,0])[:20], "cols", np.unique(np.argwhere(e > 0.5*e.max())[:,1])[:20])
