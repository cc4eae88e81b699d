"""Row-slab mode (configs 4 and 5) on ONE GPU: the device time of one rank's
block over its extended slab (its rows plus k*R neighbour rows on each side,
k sweeps per exchange) for G = 1, 2, 4, 8 ranks, and the aggregate
MPix*it/s it implies.  Two engines are timed: the resident one the product
uses (pdz_fixed_point_sweeps_resident: iterates stay in the padded layout,
the block is the persistent launch alone) and the copying one
(pdz_fixed_point_sweeps_from: pad-init + launch + extract per block).  The
ranks are independent between exchanges, so a rank's block IS its compute
time; the halo exchange cannot be measured on one GPU and is MODELLED from
the bytes it moves: 2 directions at the measured NVLink peer-copy rate
(770 GB/s per direction, B200_PROFILING.md) plus 2 x 10 us of NCCL
point-to-point launch latency per exchange; fixed-iteration runs all-reduce
the residual table once per solve (nothing per block).  Seeded synthetic
fields.
usage: python tools/slab_projection.py [--reps N]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2506_08793_b200 as pdz  # noqa: E402
from paper_2506_08793_b200 import _native as nat  # noqa: E402
from paper_2506_08793_b200.parallel import (default_sweeps_per_exchange, halo_rows,  # noqa: E402
                                            slab_bounds)
from paper_2506_08793_b200.solver import _params  # noqa: E402

TAU = 0.9 * 2.0 / (8.0 / 1e-3 + 0.5)
CONFIGS = [("config4 3840x2160 K=25", 2160, 3840, 25, 4.0, 500),
           ("config5 7680x4320 K=49", 4320, 7680, 49, 8.0, 2000)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    lib = nat.lib()
    dev = nat.device()
    base_us = {}
    for name, H, W, K, sigma, iters in CONFIGS:
        R = halo_rows(K)
        cfg = pdz.SolverConfig(tau=TAU, sigma=sigma, kernel_size=K, max_iters=iters,
                               rel_tol=1e-300)
        for G in (1, 2, 4, 8):
            rank = G // 2  # an interior rank (both halos) when G > 1
            y0, y1 = slab_bounds(H, G, rank)
            n = y1 - y0
            min_rows = min(slab_bounds(H, G, r)[1] - slab_bounds(H, G, r)[0] for r in range(G))
            k = default_sweeps_per_exchange(min_rows, R, G, iters, width=W, planes=3,
                                            kernel_size=K)
            if G == 1:
                k = 40  # a sample of the single block (the full solve is one block)
            top = min(k * R, y0) if G > 1 else 0
            bot = min(k * R, H - y1) if G > 1 else 0
            E = n + top + bot
            rng = np.random.default_rng(G)
            u = torch.from_numpy(rng.uniform(0, 1, (3, E, W)).astype(np.float32)).to(dev)
            phi = torch.from_numpy(rng.uniform(-0.2, 1.2, (3, E, W)).astype(np.float32)).to(dev)
            lam = torch.from_numpy(rng.uniform(0.02, 0.5, (E, W)).astype(np.float32)).to(dev)
            prm = _params(E, W, 3, 3, cfg, tau=TAU, max_iters=k)
            ws = torch.empty(lib.pdz_solve_workspace_bytes(prm), dtype=torch.uint8, device=dev)
            out = torch.empty_like(u)
            sums = torch.empty((k, 3), dtype=torch.float64, device=dev)
            failed = torch.empty(3, dtype=torch.int32, device=dev)
            s = torch.cuda.current_stream()

            def run_copying():
                nat.check(lib.pdz_fixed_point_sweeps_from(
                    prm, nat.ptr(u), nat.ptr(phi), nat.ptr(lam), top, top + n, nat.ptr(out),
                    nat.ptr(sums), nat.ptr(failed), nat.ptr(ws), ws.numel(), nat.stream_ptr()))

            base = [0]

            def run_resident(first=False):
                nat.check(lib.pdz_fixed_point_sweeps_resident(
                    prm, nat.ptr(u) if first else None, nat.ptr(phi), nat.ptr(lam), top, top + n,
                    base[0], nat.ptr(sums), nat.ptr(failed), nat.ptr(ws), ws.numel(),
                    nat.stream_ptr()))
                base[0] = (base[0] + k) % 3

            def timed(fn):
                for _ in range(2):
                    fn()
                torch.cuda.synchronize()
                times = []
                for _ in range(args.reps):
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                    fn()
                    e1.record(s)
                    e1.synchronize()
                    times.append(e0.elapsed_time(e1))
                return float(np.median(times))

            ms_copy = timed(run_copying)
            run_resident(first=True)
            ms = timed(run_resident)
            us_sweep = ms * 1e3 / k
            halo_bytes = (top + bot) * W * 3 * 4
            # modelled exchange per block: each direction moves its halo at the
            # measured peer-copy rate; two point-to-point launches' latency
            xchg_us = 0.0 if G == 1 else max(top, bot) * W * 3 * 4 / 770e9 * 1e6 + 2 * 10.0
            us_total = us_sweep + xchg_us / k
            if G == 1:
                base_us[name] = us_sweep
            print(json.dumps({
                "config": name, "ranks": G, "rank_rows": n, "sweeps_per_exchange": k,
                "extended_rows": E, "block_ms_resident": round(ms, 4),
                "block_ms_copying": round(ms_copy, 4),
                "us_per_sweep_compute": round(us_sweep, 2),
                "modelled_exchange_us_per_block": round(xchg_us, 1),
                "us_per_sweep_with_exchange": round(us_total, 2),
                "aggregate_mpix_it_per_s": round(H * W / 1e6 / (us_total * 1e-6)),
                "speedup_vs_one_gpu": round(base_us[name] / us_total, 2),
                "halo_bytes_per_exchange": halo_bytes,
                "kernel": int(lib.pdz_sweep_kernel_kind(prm))}), flush=True)


if __name__ == "__main__":
    main()
