"""Race hunt for the persistent sweep: solve the same problems many times,
interleaved (so buffers are reused with other problems' stale contents), and
require every repeat to be bitwise identical to the first solve and finite.
usage: python tools/stress_determinism.py [--reps N]  (PDZ_LIB_NAME selects a variant)"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2506_08793_b200 as pdz  # noqa: E402

TAU = 0.9 * 2.0 / (8.0 / 1e-3 + 0.5)
CASES = [((600, 3000), 13), ((600, 3840), 25), ((300, 7680), 49), ((400, 136), 19),
         ((333, 128), 13), ((1024, 1024), 19), ((96, 128), 13), ((5, 3), 49)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--iters", type=int, default=3)
    args = ap.parse_args()
    probs = []
    for (h, w), k in CASES:
        rng = np.random.default_rng(h + k)
        ch = rng.random((h, w)) * 0.8 + 0.1
        t = 0.3 + 0.6 * rng.random((h, w))
        cfg = pdz.SolverConfig(tau=TAU, kernel_size=k, sigma=k / 6.0, max_iters=args.iters,
                               rel_tol=1e-300)
        probs.append((f"{h}x{w} K={k}", ch, t, cfg))
    first = {}
    bad = 0
    for rep in range(args.reps):
        for name, ch, t, cfg in probs:
            try:
                u, tr = pdz.fixed_point_solve(ch, t, 0.9, cfg)
            except Exception as e:  # noqa: BLE001
                print(f"rep {rep} {name}: {type(e).__name__}: {e}", flush=True)
                bad += 1
                continue
            key = (u.tobytes(), tuple(tr.residual_norms))
            if name not in first:
                first[name] = key
            elif key != first[name]:
                d = np.max(np.abs(np.frombuffer(key[0]) - np.frombuffer(first[name][0])))
                print(f"rep {rep} {name}: differs from the first solve (max {d:.3e})", flush=True)
                bad += 1
    print(f"stress: {args.reps} reps x {len(probs)} problems, {bad} bad", flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
