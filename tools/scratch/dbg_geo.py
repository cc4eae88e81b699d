import sys, os, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_2506_08793_b200 as pdz
from paper_2506_08793_b200 import synthetic as SYN
from conftest import TAU_STABLE
FLAGS = ("no-multiscale", "no-guided")
c = SYN.BENCH_CONFIGS[3]
imgs = [SYN.make_hazy_scene(480, 640, 3, i).hazy.astype(np.float64) for i in range(16)]
cfg = pdz.SolverConfig(tau=TAU_STABLE, sigma=c["sigma"], kernel_size=c["kernel_size"], patch_radius=c["patch_radius"], max_iters=1, rel_tol=1e-300)
res = {}
for geo in ("0", "1"):
    os.environ["PDZ_STREAM_GEO"] = geo
    res["batch", geo] = pdz.dehaze_batch(imgs, cfg, ablation=FLAGS)[0][0]
    res["single", geo] = pdz.dehaze(imgs[0], cfg, ablation=FLAGS)[0]
    os.environ["PDZ_STREAM_K"] = "1"
    res["singleK1", geo] = pdz.dehaze(imgs[0], cfg, ablation=FLAGS)[0]
    del os.environ["PDZ_STREAM_K"]
keys = list(res)
for i in range(len(keys)):
    for j in range(i + 1, len(keys)):
        d = res[keys[i]] != res[keys[j]]
        ys = np.argwhere(d)
        print(keys[i], keys[j], int(d.sum()), (ys[:8].tolist() if len(ys) else ""))
