import sys, os, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_2506_08793_b200 as pdz
from paper_2506_08793_b200 import synthetic as SYN
from conftest import TAU_STABLE
FLAGS = ("no-multiscale", "no-guided")
c = SYN.BENCH_CONFIGS[3]
img = SYN.make_hazy_scene(480, 640, 3, 0).hazy.astype(np.float64)
cfg = pdz.SolverConfig(tau=TAU_STABLE, sigma=c["sigma"], kernel_size=13, patch_radius=c["patch_radius"], max_iters=1, rel_tol=1e-300)
a = pdz.dehaze(img, cfg, ablation=FLAGS)[0]
os.environ["PDZ_STREAM_K"] = "1"
b = pdz.dehaze(img, cfg, ablation=FLAGS)[0]
d = np.argwhere(a != b)
rows = d[:, 0]
bounds = [(480*i)//14 for i in range(15)]
rel = np.array([r - max(bb for bb in bounds if bb <= r) for r in rows]) if len(d) else np.array([], dtype=int)
print(os.environ.get("PDZ_LIB_NAME"), "mism", len(d), "offset mod 6", np.bincount(rel % 6, minlength=6) if len(d) else "")
