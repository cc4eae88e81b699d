import sys, os, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_2506_08793_b200 as pdz
from paper_2506_08793_b200 import synthetic as SYN
from conftest import TAU_STABLE
FLAGS = ("no-multiscale", "no-guided")
c = SYN.BENCH_CONFIGS[3]
img = SYN.make_hazy_scene(480, 640, 3, 0).hazy.astype(np.float64)
for edge in (True, False):
  for ks in (13, 1):
    cfg = pdz.SolverConfig(tau=TAU_STABLE, sigma=c["sigma"], kernel_size=ks, patch_radius=c["patch_radius"], max_iters=1, rel_tol=1e-300)
    fl = FLAGS if edge else FLAGS + ("no-edge",)
    a = pdz.dehaze(img, cfg, ablation=fl)[0]
    os.environ["PDZ_STREAM_K"] = "1"
    b = pdz.dehaze(img, cfg, ablation=fl)[0]
    del os.environ["PDZ_STREAM_K"]
    d = np.argwhere(a != b)
    print("edge", edge, "K", ks, "mism", len(d))
    if len(d):
        rows = d[:, 0]
        print("  rows mod 6 (K1 plan: row%114%6):", np.bincount((rows % 114) % 6, minlength=6))
        # default plan: 14 CTAs per strip: boundaries
        bounds = [ (480*i)//14 for i in range(15)]
        rel = np.array([r - max(b for b in bounds if b <= r) for r in rows])
        print("  row offset within default CTA range, mod 6:", np.bincount(rel % 6, minlength=6), "offset hist", np.bincount(rel, minlength=36))
        print("  col mod 2:", np.bincount(d[:,1] % 2), "col mod 64 hist (8 bins)", np.histogram(d[:,1] % 64, bins=8)[0], "chan", np.bincount(d[:,2]))
        for (y,x,ch) in d[:5]: print("   ", y, x, ch, repr(a[y,x,ch]), repr(b[y,x,ch]))
