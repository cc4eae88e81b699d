import sys; sys.path.insert(0, '.')
import torch, ctypes
import paper_2506_08793_b200 as pdz
from paper_2506_08793_b200 import _native as nat
from paper_2506_08793_b200.solver import _params
cfg = pdz.SolverConfig(tau=2.2e-4, sigma=3.0, kernel_size=19, max_iters=20, rel_tol=1e-300)
prm = _params(1024, 1024, 3, 3, cfg)
lib = nat.lib()
print("kind", lib.pdz_sweep_kernel_kind(prm), "err", lib.pdz_last_error())
