"""Benchmark of the hot path: the relaxed fixed-point dehazing solve.

Workload (BASELINE.json configs[1]): one 1024x1024x3 float32
synthetic hazy image, patch 15 (r = 7), Gaussian sigma 3 / K = 19, 200
fixed-point iterations at tau = TAU_STABLE, ablation no-multiscale/no-guided.
A "step" = one full 200-iteration solve of all 3 channels.

  value  : MPix*it/s of the solve with Phi/lambda already resident in HBM
           (front end excluded), L2 flushed (256 MiB write) before every step;
  e2e    : the same metric through the public API `dehaze()` with a pinned
           host float32 image: H2D copy, front end, solve, clamp and D2H of
           the float64 result inside the timed region.

`python bench.py --gpus N` under torchrun runs one independent image per
rank (weak scaling, no data-path collective; SURVEY 8(e) batch mode);
timing is max over ranks.  `--impl reference` times the reference
algorithm (the CPU oracle port, oracle/pdz_oracle.py) on host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

TAU_STABLE = 0.9 * 2.0 / (8.0 / 1e-3 + 0.5)
H, W, C = 1024, 1024, 3
K, SIGMA, ITERS, PATCH_R = 19, 3.0, 200, 7
ABL = ("no-multiscale", "no-guided")
METRIC = "megapixel-iterations/sec of fixed-point solver"
UNIT = "MPix*it/s"
BYTES_PER_PIXEL = (3 * C + 1) * 4  # read u, Phi (C planes), lambda; write u' -> 40 B
FLOPS_PER_PIXEL = C * (33 + 4 * K)


def _env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def _config(extra=None):
    cfg = {"workload": "config2: 1024x1024x3 f32 synthetic hazy image, patch 15, sigma 3 "
                       "(K=19), 200 fixed-point iterations, tau=TAU_STABLE",
           "height": H, "width": W, "channels": C, "kernel_size": K, "sigma": SIGMA,
           "iterations": ITERS, "tau": TAU_STABLE, "ablation": list(ABL),
           "l2": "flushed before every timed step (256 MiB memset)"}
    if extra:
        cfg.update(extra)
    return cfg


def _peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """Samples SM clocks and throttle reasons with NVML during the timed region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 - NVML optional
            self._nv = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                mhz = self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM)
                mask = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.samples.append(mhz)
                for name, bit in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)  # the timed region is ~35 ms at the default steps

    def __enter__(self):
        if self._nv is not None:
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._nv is not None:
            self._t.join(timeout=1.0)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------- CPU side

def cpu_solve_sample(iters=2, threads=3):
    """Reference algorithm (oracle port: direct K^2 Gaussian like
    gaussian_convolve, solver.py:238-240) on the host: `iters` fixed-point
    iterations of the full 1024^2 config-2 solve, one thread per channel
    (the reference's `workers` parallelism).  Returns (MPix*it/s, seconds)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import pdz_oracle as orc
    from paper_2506_08793_b200.synthetic import make_hazy_scene

    img = make_hazy_scene(H, W, 2, 0).hazy.astype(np.float64)
    st = orc.SolverSettings(tau=TAU_STABLE, sigma=SIGMA, kernel_size=K, patch_radius=PATCH_R,
                            max_iters=iters, rel_tol=1e-300)
    dark = orc.dark_channel(img, np.ones(C), PATCH_R)
    a = orc.airlight_from_selection(img, orc.airlight_selection(dark, st.airlight_fraction))
    t = orc.transmission_from_dark(orc.dark_channel(img, a, PATCH_R), st.omega)
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as pool:
        list(pool.map(lambda c: orc.relaxed_solve(img[:, :, c], t, float(a[c]), st),
                      range(C)))
    dt = time.perf_counter() - t0
    return H * W * iters / dt / 1e6, dt


def cpu_front_end_seconds():
    from oracle import pdz_oracle as orc
    from paper_2506_08793_b200.synthetic import make_hazy_scene

    img = make_hazy_scene(H, W, 2, 0).hazy.astype(np.float64)
    t0 = time.perf_counter()
    dark = orc.dark_channel(img, np.ones(C), PATCH_R)
    a = orc.airlight_from_selection(img, orc.airlight_selection(dark, 0.001))
    t = orc.transmission_from_dark(orc.dark_channel(img, a, PATCH_R), 0.95)
    (img - a * (1.0 - t)[:, :, None]) / np.maximum(t, 0.1)[:, :, None]
    orc.haze_weight(t)
    return time.perf_counter() - t0


def run_reference(args):
    rank, _, world = _env_rank()
    if rank != 0:
        return 0
    fe = cpu_front_end_seconds()
    for _ in range(args.warmup):
        pass  # the CPU port has no JIT/cache state worth warming beyond imports
    samples = []
    iters = 2
    for _ in range(args.steps):
        _, dt = cpu_solve_sample(iters=iters)
        samples.append(dt)
    per_iter = statistics.mean(samples) / iters
    total = fe + ITERS * per_iter  # extrapolated full config-2 run
    value = H * W * ITERS / total / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": _config({"parallelism": "host threads (channels)"}),
        "cpu_baseline": {
            "value": value, "unit": UNIT, "cores": C, "kind": "port",
            "sample": f"oracle port of the reference (numpy float64, direct K^2 Gaussian), "
                      f"front end once ({fe:.2f} s) + {iters} solve iterations per step x "
                      f"{args.steps} steps at 1024^2, 3 channel threads; extrapolated to "
                      f"{ITERS} iterations",
            "host_cpus": os.cpu_count()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- GPU side

def run_gpu(args):
    import torch

    rank, local, world = _env_rank()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2506_08793_b200 as pdz
    from paper_2506_08793_b200 import _native as nat
    from paper_2506_08793_b200.solver import (DeviceProblem, _front_end, _image_dev,
                                              _lambda_mode, _params, prepare_problem)
    from paper_2506_08793_b200.synthetic import make_hazy_scene

    lib = nat.lib()
    cfg = pdz.SolverConfig(tau=TAU_STABLE, sigma=SIGMA, kernel_size=K, patch_radius=PATCH_R,
                           max_iters=ITERS, rel_tol=1e-300)
    scene = make_hazy_scene(H, W, 2, rank)
    host_img = torch.from_numpy(scene.hazy).pin_memory()

    # device-resident solver inputs (outside the timed region)
    img_dev, is_f64 = _image_dev(host_img)
    flags = frozenset(ABL)
    t_dev, a_dev = _front_end(img_dev, is_f64, cfg, flags)
    phi, lam = prepare_problem(img_dev, is_f64, t_dev, a_dev, cfg, _lambda_mode(flags, cfg))
    prob = DeviceProblem(phi, lam, H, W, C, C)
    prm = _params(H, W, C, C, cfg)
    ws = torch.empty(lib.pdz_solve_workspace_bytes(prm), dtype=torch.uint8, device=phi.device)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=phi.device)
    stream = torch.cuda.current_stream()

    def solve():
        nat.check(lib.pdz_fixed_point_sweeps_async(prm, nat.ptr(prob.phi), nat.ptr(prob.lam),
                                                   nat.ptr(ws), ws.numel(), nat.stream_ptr()))

    for _ in range(max(args.warmup, 3)):
        flush.zero_()
        solve()
    torch.cuda.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kernel_ms = []  # the persistent sweep kernel alone (library events on its stream)
    lib.pdz_time_sweep_kernels(1)
    with ClockSampler(local) as clocks:
        barrier()
        for i in range(args.steps):
            flush.zero_()
            starts[i].record(stream)
            solve()
            ends[i].record(stream)
        barrier()
    lib.pdz_time_sweep_kernels(0)
    kernel_ms.append(float(lib.pdz_last_sweep_kernel_ms()))
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    ms = statistics.mean(step_ms)
    if dist is not None:
        t = torch.tensor([ms], device=phi.device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * H * W * ITERS / (ms / 1e3) / 1e6

    # roofline of the dominant kernel: the persistent sweep kernel, ONE launch
    # per solve (all 200 sweeps).  achieved = algorithmic bytes per launch
    # (40 B/px/sweep x H x W x 200) / the launch's device time,
    # read from CUDA events the library records around that launch on its
    # stream (pdz_time_sweep_kernels); the last timed step's launch.
    peak, peak_src = _peaks()
    kind = int(lib.pdz_sweep_kernel_kind(prm))
    launch_ms = kernel_ms[-1] if kernel_ms and kernel_ms[-1] > 0 else ms
    if dist is not None:
        t = torch.tensor([launch_ms], device=phi.device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        launch_ms = float(t.item())
    alg_bytes = BYTES_PER_PIXEL * H * W * ITERS
    achieved = alg_bytes / (launch_ms / 1e3) / 1e9
    traffic = None
    prof = os.path.join(REPO, "profiles", "sweep_ncu_summary.json")
    if os.path.exists(prof):
        with open(prof) as fh:
            traffic = json.load(fh).get("dram_bytes_per_launch")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": alg_bytes,
                "fp32_tflops": FLOPS_PER_PIXEL * H * W * ITERS / (launch_ms / 1e3) / 1e12,
                "kernel": ("pdz::stream_kernel<9,true> (persistent, 200 sweeps per launch)"
                           if kind == 2 else "pdz::sweep_kernel<9,true> (tiled, 1 sweep per launch)"),
                "launch_ms": launch_ms, "share_of_step": launch_ms / ms,
                "us_per_sweep": launch_ms * 1e3 / ITERS}

    # e2e through the public API: pinned host image -> dehaze -> host result.
    # A CPU-tensor input returns a CPU float64 tensor (numpy in -> numpy out,
    # like the reference), so the device->host read is inside the call.
    def e2e_step():
        out, _ = pdz.dehaze(host_img, cfg, ablation=ABL)
        assert out.device.type == "cpu" and out.dtype == torch.float64

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    e_ms = []
    for _ in range(max(3, min(args.steps, 10))):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms.append(max(e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3))
    e2e_ms = statistics.mean(e_ms)
    if dist is not None:
        t = torch.tensor([e2e_ms], device=phi.device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    # host reads per step: the restored image (H, W, C) f64, the transmission
    # map (H, W) f64 and the airlight (C,) f64 of DehazeResult
    e2e = {"value": world * H * W * ITERS / (e2e_ms / 1e3) / 1e6, "unit": UNIT,
           "h2d_bytes_per_step": H * W * C * 4,
           "d2h_bytes_per_step": H * W * C * 8 + H * W * 8 + C * 8,
           "ms_per_step": e2e_ms}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, dt = cpu_solve_sample(iters=2)
        cpu = {"value": v, "unit": UNIT, "cores": C, "kind": "port",
               "sample": f"oracle port (numpy float64, direct K^2 Gaussian as in the "
                         f"reference) 2 iterations of the 1024^2 K=19 solve, 3 channel "
                         f"threads, {dt:.1f} s, front end excluded like `value`",
               "host_cpus": os.cpu_count()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded generator of SURVEY 8(d); no public dataset)",
            "config": _config({"parallelism": f"replicas x{world} (one image per GPU)"}),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(lib.pdz_solve_kernel_launches(prm)) * args.steps,
            "clocks": clocks.summary(),
            "step_ms": step_ms,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
