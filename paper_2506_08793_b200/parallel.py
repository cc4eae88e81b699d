"""Multi-GPU modes of the hot path.

Batch mode (config 3) needs no collective: every rank dehazes its own images
(`dehaze_batch`; `bench.py --config 3 --gpus N` deals ceil(256 / N) images to
each rank).

Row-slab mode (configs 4 and 5, one large image) is implemented here:

* every rank runs the (cheap, < 1 %) front end on the whole image, so all
  ranks hold identical Phi, lambda and tau bounds;
* rank k owns the global rows [y0, y1) = slab_bounds(H, G, k) of ALL C
  planes;
* the solve advances in BLOCKS of k sweeps (temporal blocking): before a
  block (except the first: u0 = Phi is known everywhere) the ranks exchange
  k*R rows with each neighbour (torch.distributed point-to-point: NCCL on
  GPUs, gloo in the CPU tests), R = max(1, K // 2), so each rank holds an
  extended slab of its rows plus up to k*R neighbour rows on each side.  One
  sweep moves information R rows, so after n <= k sweeps of the extended
  slab treated as an image of its own (rows 0 / E-1 as image borders:
  exactly the global borders at the top of rank 0 and the bottom of rank
  G-1, fake ones elsewhere) the rank's own rows are exact -- bit for bit the
  whole-image arithmetic;
* a block runs on the device as ONE persistent-kernel launch, and the
  slab's iterates stay RESIDENT in the kernel's padded layout for the whole
  solve (pdz_fixed_point_sweeps_resident, include/pdz.h): the block starts
  from the buffer the previous one ended in, and the halo exchange writes
  the received rows straight into that buffer through a strided view -- no
  copy into or out of the padded layout per block;
* fixed-iteration runs (rel_tol < DEFERRED_TOL) never wait for the host: the
  per-sweep sums of r^2 collect in a device table [iters][C] that is
  all-reduced ONCE at the end.  With a real tolerance the [k][C] table is
  all-reduced per block and every rank applies the same global stop rule
  (solver.py:347-358) to the k sweeps in order; a plane that stopped inside
  a block takes the iterate after its stopping sweep, recomputed from the
  block's start (kept only on that path);
* the final slabs are all-gathered into the full image on every rank.

k trades the redundant halo sweeps (2kR rows per block) against one
exchange + launch per block; the default is min(4, slab rows // R) (the 2-4
sweeps per launch of the north star; tools/slab_projection.py measures a
rank's block on one GPU and models the exchange).  The engine is pluggable
(`block=`) so the CPU tests drive the same host logic with an oracle engine
on CPU tensors; the default engine is the CUDA one and there is no CPU
fallback in the product.
"""

from __future__ import annotations

import logging
import math

from . import _native as nat
from .config import DehazeResult, SolverConfig, SolverTrace, normalize_ablation
from .image import to_host, validate_image

logger = logging.getLogger("pdehaze.solver")

__all__ = ["slab_bounds", "halo_rows", "default_sweeps_per_exchange", "SlabSolver",
           "solve_slab", "dehaze_slabs"]


def slab_bounds(height: int, world: int, rank: int) -> tuple[int, int]:
    """Global rows [y0, y1) of rank `rank`: ceil(H / G) rows each, the last
    rank takes the remainder."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside a world of {world}")
    rows = -(-height // world)
    y0 = min(height, rank * rows)
    return y0, min(height, y0 + rows)


def halo_rows(kernel_size: int) -> int:
    """Halo depth of one sweep: the Gaussian radius K // 2, and at least the
    one row the divergence stencil needs."""
    return max(1, kernel_size // 2)


def _global_rank(group, r):
    import torch.distributed as dist

    return r if group is None else dist.get_global_rank(group, r)


class _FunctionalEngine:
    """Slab iterate held as a dense tensor and advanced by a pure block
    function `block(u, phi_e, lam_e, lo, hi, n) -> (u_new, sums [n][P], failed
    [P])`.  The CPU tests plug the oracle in here (gloo ranks on CPU tensors);
    the product uses _ResidentEngine."""

    def __init__(self, block, phi_e, lam_e, lo, hi):
        self.block, self.phi_e, self.lam_e, self.lo, self.hi = block, phi_e, lam_e, lo, hi
        self.u = phi_e.clone()  # u0 = Phi (solver.py:333)
        self.start = None

    def field(self):
        return self.u

    def run(self, n, keep_start):
        self.start = self.u if keep_start else None
        self.u, sums, failed = self.block(self.u, self.phi_e, self.lam_e, self.lo, self.hi, n)
        return sums, failed

    def after(self, s):
        """Iterate after `s` sweeps of the last block (started with keep_start)."""
        return self.block(self.start, self.phi_e, self.lam_e, self.lo, self.hi, s)[0]

    def reset(self):
        self.u = self.phi_e.clone()


class _ResidentEngine:
    """The product engine: the slab's iterates stay in the padded layout of the
    persistent kernel inside one workspace for the whole solve
    (pdz_fixed_point_sweeps_resident).  A block is one persistent launch that
    starts from the buffer the previous block ended in; `field()` is a strided
    view of that buffer's field, so the halo exchange writes the k*R neighbour
    rows straight into it -- no copy into or out of the padded layout per
    block."""

    def __init__(self, cfg, tau, edge_preserving, phi_e, lam_e, lo, hi, kmax):
        import numpy as np
        import torch

        from .solver import _params

        self.lib = nat.lib()
        self.phi_e, self.lam_e, self.lo, self.hi = phi_e, lam_e, int(lo), int(hi)
        self.planes, self.rows, self.width = phi_e.shape
        self._prm = lambda n: _params(self.rows, self.width, self.planes, self.planes, cfg,
                                      edge_preserving=edge_preserving, tau=tau, max_iters=n)
        prm = self._prm(kmax)
        # a private workspace: it carries the iterates from block to block
        self.ws = torch.empty(int(self.lib.pdz_solve_workspace_bytes(prm)), dtype=torch.uint8,
                              device=phi_e.device)
        info = np.zeros(8, dtype=np.int64)
        nat.check(self.lib.pdz_slab_layout(prm, info.ctypes.data, 8))
        self.nbuf, pr, pc, hp, wp = int(info[0]), int(info[4]), int(info[5]), int(info[6]), \
            int(info[7])
        nbytes = self.planes * hp * wp * 4
        self.fields = []
        for b in range(self.nbuf):
            padded = self.ws[int(info[1 + b]):int(info[1 + b]) + nbytes].view(torch.float32)
            self.fields.append(padded.view(self.planes, hp, wp)[:, pr:pr + self.rows,
                                                                pc:pc + self.width])
        self.cur = 0          # buffer holding the current iterate
        self.fresh = True     # before the first block the iterate is u0 = Phi itself
        self.start = None

    def field(self):
        return self.phi_e if self.fresh else self.fields[self.cur]

    def run(self, n, keep_start):
        import torch

        if keep_start:
            self.start = self.phi_e if self.fresh else self.fields[self.cur].clone()
        else:
            self.start = None
        sums = torch.empty((n, self.planes), dtype=torch.float64, device=self.ws.device)
        failed = torch.empty(self.planes, dtype=torch.int32, device=self.ws.device)
        # the first block loads u0 = Phi into buffer 0 (and poisons every pad)
        u_init = nat.ptr(self.phi_e) if self.fresh else None
        nat.check(self.lib.pdz_fixed_point_sweeps_resident(
            self._prm(n), u_init, nat.ptr(self.phi_e), nat.ptr(self.lam_e), self.lo, self.hi,
            self.cur, nat.ptr(sums), nat.ptr(failed), nat.ptr(self.ws), self.ws.numel(),
            nat.stream_ptr()))
        self.fresh = False
        self.cur = (self.cur + n) % self.nbuf
        return sums, failed

    def after(self, s):
        import torch

        prm = self._prm(s)
        ws = nat.workspace(self.lib.pdz_solve_workspace_bytes(prm), "slab-redo")
        out = torch.empty_like(self.start)
        sums = torch.empty((s, self.planes), dtype=torch.float64, device=out.device)
        failed = torch.empty(self.planes, dtype=torch.int32, device=out.device)
        nat.check(self.lib.pdz_fixed_point_sweeps_from(
            prm, nat.ptr(self.start), nat.ptr(self.phi_e), nat.ptr(self.lam_e), self.lo, self.hi,
            nat.ptr(out), nat.ptr(sums), nat.ptr(failed), nat.ptr(ws), ws.numel(),
            nat.stream_ptr()))
        return out

    def reset(self):
        self.fresh, self.cur = True, 0


# Cost model behind the default k (microseconds; B200, measured in
# profiles/r2_slab_projection.jsonl and B200_PROFILING.md): the sweep kernel
# sustains ~26 TFLOP/s of its C * (33 + 4K) FLOP per pixel, a block costs one
# persistent launch plus two small init launches, and an exchange costs two
# NCCL point-to-point launches plus its bytes at the NVLink peer-copy rate.
_SWEEP_TFLOPS = 26.0
_BLOCK_LAUNCH_US = 26.0  # ~7 us of launches around + ~19 us pipeline fill / drain inside
_EXCHANGE_LATENCY_US = 20.0
_NVLINK_BYTES_PER_US = 770e3


def default_sweeps_per_exchange(min_rows: int, halo: int, world: int, max_iters: int,
                                width: int | None = None, planes: int = 3,
                                kernel_size: int | None = None) -> int:
    """k of the temporal blocking: one block for a single rank; else at most
    4 sweeps (the north star's 2-4 per launch) and never deeper than a
    neighbour's slab (k*R <= its rows).  With the slab's `width` and
    `kernel_size` given, k in 1..4 minimises the modelled time per sweep,
    (rows + 2kR) * row cost + (launch + exchange latency + 2kR-row bytes) / k:
    deeper blocks amortise the exchange but sweep 2kR redundant rows."""
    if world == 1:
        return max(1, max_iters)
    kmax = max(1, min(4, min_rows // halo, max_iters))
    if width is None or kernel_size is None:
        return kmax
    row_us = width * planes * (33 + 4 * kernel_size) / (_SWEEP_TFLOPS * 1e6)
    row_bytes = width * planes * 4

    def per_sweep(k):
        exchange = _EXCHANGE_LATENCY_US + k * halo * row_bytes / _NVLINK_BYTES_PER_US
        return (min_rows + 2 * k * halo) * row_us + (_BLOCK_LAUNCH_US + exchange) / k

    return min(range(1, kmax + 1), key=per_sweep)


#: rel_tol below this can only stop a plane whose residual norm repeats
#: exactly; such runs ("fixed iteration count") take the deferred path
DEFERRED_TOL = 1e-12


class SlabSolver:
    """One rank's share of a row-slab solve.

    phi: (C, H, W) full Phi (every rank holds it after the replicated front
    end); lam: (H, W).  `sweeps_per_exchange` = k of the temporal blocking
    (default: default_sweeps_per_exchange).
    """

    def __init__(self, phi, lam, height: int, cfg: SolverConfig, *, tau: float,
                 edge_preserving: bool = True, group=None, rank: int = 0, world: int = 1,
                 block=None, sweeps_per_exchange: int | None = None):
        self.cfg, self.tau, self.height = cfg, float(tau), int(height)
        self.group, self.rank, self.world = group, rank, world
        self.y0, self.y1 = slab_bounds(self.height, world, rank)
        self.rows = self.y1 - self.y0
        self.halo = R = halo_rows(cfg.kernel_size)
        min_rows = min(slab_bounds(self.height, world, k)[1] - slab_bounds(self.height, world, k)[0]
                       for k in range(world))
        if min_rows < R:
            raise ValueError(f"{world} row slabs of a {self.height}-row image leave fewer than "
                             f"the {R} halo rows per slab")
        k = sweeps_per_exchange or default_sweeps_per_exchange(
            min_rows, R, world, cfg.max_iters, width=int(phi.shape[2]), planes=int(phi.shape[0]),
            kernel_size=cfg.kernel_size)
        if world > 1 and k * R > min_rows:
            raise ValueError(f"{k} sweeps per exchange need {k * R} halo rows, more than the "
                             f"{min_rows} rows of the thinnest slab")
        self.k = int(k)
        depth = self.k * R if world > 1 else 0
        self.top = min(depth, self.y0)                  # neighbour rows above
        self.bot = min(depth, self.height - self.y1)    # and below
        a, b = self.y0 - self.top, self.y1 + self.bot   # global rows of the extended slab
        self.planes, self.width = phi.shape[0], phi.shape[2]
        self.phi_e = phi[:, a:b].contiguous().clone()
        self.lam_e = lam[a:b].contiguous().clone()
        t, n = self.top, self.rows
        if block is None:
            self.engine = _ResidentEngine(cfg, self.tau, edge_preserving, self.phi_e, self.lam_e,
                                          t, t + n, min(self.k, cfg.max_iters))
        else:
            self.engine = _FunctionalEngine(block, self.phi_e, self.lam_e, t, t + n)

    @property
    def u(self):
        """The current extended-slab iterate (C, E, W)."""
        return self.engine.field()

    # -- halo exchange -----------------------------------------------------
    def exchange(self, u):
        """Fill the neighbour rows of the extended slab `u` (C, E, W; possibly
        a strided view of the resident iterate) with the neighbours' current
        rows."""
        if self.world == 1 or (self.top == 0 and self.bot == 0):
            return
        import torch
        import torch.distributed as dist

        t, n = self.top, self.rows
        ops, recv = [], {}
        if self.rank > 0:
            peer = _global_rank(self.group, self.rank - 1)
            # the rank above holds `t` rows of ours below its slab
            ops.append(dist.P2POp(dist.isend, u[:, t:t + t].contiguous(), peer, self.group))
            recv["top"] = torch.empty((u.shape[0], t, u.shape[2]), dtype=u.dtype, device=u.device)
            ops.append(dist.P2POp(dist.irecv, recv["top"], peer, self.group))
        if self.rank < self.world - 1:
            peer = _global_rank(self.group, self.rank + 1)
            b = self.bot
            ops.append(dist.P2POp(dist.isend, u[:, t + n - b:t + n].contiguous(), peer,
                                  self.group))
            recv["bot"] = torch.empty((u.shape[0], b, u.shape[2]), dtype=u.dtype, device=u.device)
            ops.append(dist.P2POp(dist.irecv, recv["bot"], peer, self.group))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        if "top" in recv:
            u[:, :t] = recv["top"]
        if "bot" in recv:
            u[:, t + n:] = recv["bot"]

    def _allreduce(self, sums, failed):
        if self.world > 1:
            import torch
            import torch.distributed as dist

            dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=self.group)
            big = torch.iinfo(torch.int32).max
            first = torch.where(failed > 0, failed, torch.full_like(failed, big))
            dist.all_reduce(first, op=dist.ReduceOp.MIN, group=self.group)
            failed = torch.where(first == big, torch.zeros_like(first), first)
        return sums, failed

    # -- the solve -----------------------------------------------------------
    def solve(self, max_iters: int, rel_tol: float):
        """fixed_point_solve (solver.py:343-358) of every plane over the slab.
        Returns (u slab (C, y1 - y0, W), norms [C] lists, iterations [C],
        converged [C]).

        rel_tol < DEFERRED_TOL ("fixed iteration count"): no block waits for
        the host -- the per-sweep sums of r^2 collect in a device table
        [max_iters][C] that is all-reduced ONCE at the end, and the stop rule
        runs over the finished table; should a plane's norm ever repeat
        exactly (the only way such a tolerance stops early), the solve is
        redone on the per-block path below, which is exact for any rel_tol."""
        if rel_tol < DEFERRED_TOL:
            done = self._solve_deferred(max_iters, rel_tol)
            if done is not None:
                return done
            self.engine.reset()
        return self._solve_per_block(max_iters, rel_tol)

    def _solve_deferred(self, max_iters, rel_tol):
        import torch

        t, n, P = self.top, self.rows, self.planes
        eng = self.engine
        table, bad = [], None
        it = 0
        while it < max_iters:
            k = min(self.k, max_iters - it)
            if it:  # u0 = Phi: every rank already holds its halo rows of it
                with nat.trace_range("pdz.slab.exchange"):
                    self.exchange(eng.field())
            with nat.trace_range("pdz.slab.block"):
                sums, failed = eng.run(k, keep_start=False)
            table.append(sums)
            first = torch.where(failed > 0, failed + it, torch.zeros_like(failed))
            bad = first if bad is None else torch.where(bad > 0, bad, first)
            it += k
        sums, bad = self._allreduce(torch.cat(table, dim=0), bad)
        sums_h, bad_h = sums.to("cpu").numpy(), bad.to("cpu").numpy()
        norms = [[] for _ in range(P)]
        for p in range(P):
            prev = None
            for s in range(1, max_iters + 1):
                if 0 < bad_h[p] <= s:
                    raise FloatingPointError(
                        f"solver produced non-finite values at iteration {s}")
                nrm = math.sqrt(float(sums_h[s - 1, p]))
                norms[p].append(nrm)
                if prev is not None and abs(nrm - prev) / max(prev, 1e-30) <= rel_tol \
                        and s < max_iters:
                    return None  # an exact repeat: take the per-block path
                prev = nrm
        conv = []
        for p in range(P):
            last, before = norms[p][-1], (norms[p][-2] if max_iters > 1 else None)
            conv.append(before is not None and abs(last - before) / max(before, 1e-30) <= rel_tol)
        result = eng.field()[:, t:t + n].clone()
        return result, norms, [max_iters] * P, conv

    def _solve_per_block(self, max_iters, rel_tol):
        t, n = self.top, self.rows
        P = self.planes
        eng = self.engine
        result = eng.field()[:, t:t + n].clone()
        running = [True] * P
        prev = [None] * P
        norms = [[] for _ in range(P)]
        iters = [0] * P
        conv = [False] * P
        it = 0
        while it < max_iters and any(running):
            k = min(self.k, max_iters - it)
            if it:
                with nat.trace_range("pdz.slab.exchange"):
                    self.exchange(eng.field())
            with nat.trace_range("pdz.slab.block"):
                sums, failed = eng.run(k, keep_start=True)
            sums, failed = self._allreduce(sums, failed)
            sums_h = sums.to("cpu").numpy()
            failed_h = failed.to("cpu").numpy()
            stop_at = {}
            for s in range(1, k + 1):
                for p in range(P):
                    if not running[p]:
                        continue
                    if 0 < failed_h[p] <= s:
                        raise FloatingPointError(
                            f"solver produced non-finite values at iteration {it + s}")
                    nrm = math.sqrt(float(sums_h[s - 1, p]))
                    norms[p].append(nrm)
                    iters[p] = it + s
                    stop = False
                    if prev[p] is not None and abs(nrm - prev[p]) / max(prev[p], 1e-30) <= rel_tol:
                        conv[p] = stop = True
                    elif it + s >= max_iters:
                        stop = True
                    prev[p] = nrm
                    if stop:
                        running[p] = False
                        stop_at[p] = s
            # the answer is the iterate after the stopping update: recomputed
            # from the block's start for a plane that stopped inside the block
            for s in sorted(set(stop_at.values())):
                u_s = eng.field() if s == k else eng.after(s)
                for p, sp in stop_at.items():
                    if sp == s:
                        result[p] = u_s[p, t:t + n]
            it += k
        return result, norms, iters, conv


def solve_slab(phi, lam, height, cfg: SolverConfig, *, tau=None, edge_preserving=True,
               bounds=None, group=None, block=None, sweeps_per_exchange=None, warn=True):
    """Row-slab fixed_point_solve of all C planes on the calling rank.
    Returns (u slab (C, rows, W), [SolverTrace] * C) -- the traces (global
    norms) are identical on every rank."""
    rank, world = 0, 1
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            rank, world = dist.get_rank(group), dist.get_world_size(group)
    except ImportError:  # pragma: no cover - torch always ships distributed here
        pass
    step_size = cfg.tau if tau is None else float(tau)
    if warn and bounds is not None and rank == 0:
        for b in bounds:
            if step_size > b:
                logger.warning(
                    "relaxation step %.3g exceeds the stability bound %.3g at the "
                    "initial iterate; convergence is not guaranteed", step_size, b)
    solver = SlabSolver(phi, lam, height, cfg, tau=step_size, edge_preserving=edge_preserving,
                        group=group, rank=rank, world=world, block=block,
                        sweeps_per_exchange=sweeps_per_exchange)
    u, norms, iters, conv = solver.solve(cfg.max_iters, cfg.rel_tol)
    bl = list(bounds) if bounds is not None else [float("nan")] * solver.planes
    traces = [SolverTrace(residual_norms=norms[p], iterations_run=iters[p], converged=conv[p],
                          tau_used=step_size, tau_bound=float(bl[p]))
              for p in range(solver.planes)]
    return u, traces


def _all_gather_rows(slab, height, group, rank, world):
    """Concatenate every rank's rows (C, rows_k, W) into (C, H, W)."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return slab
    rows = -(-height // world)
    pad = torch.zeros((slab.shape[0], rows, slab.shape[2]), dtype=slab.dtype,
                      device=slab.device)
    pad[:, :slab.shape[1]] = slab
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    out = [parts[k][:, :slab_bounds(height, world, k)[1] - slab_bounds(height, world, k)[0]]
           for k in range(world)]
    return torch.cat(out, dim=1)


def dehaze_slabs(image, cfg: SolverConfig | None = None, ablation=(), group=None):
    """`dehaze` (solver.py:375-436) of ONE image split into row slabs over the
    ranks of `group` (one GPU per rank, torch.distributed initialised with
    NCCL).  Every rank returns the full restored image and DehazeResult."""
    import torch
    import torch.distributed as dist

    from .solver import (_front_end, _image_dev, _lambda_mode, _unit_range, prepare_problem)

    cfg = cfg or SolverConfig()
    flags = normalize_ablation(ablation)
    if "no-pde" in flags:
        from .solver import dehaze

        return dehaze(image, cfg, ablation)
    img = validate_image(image)
    _unit_range(img)
    img_dev, is_f64 = _image_dev(img)
    h, w, c = img_dev.shape
    if h < 2 or w < 2:
        raise ValueError(f"field must be at least 2x2, got {(h, w)}")
    t_dev, a_dev = _front_end(img_dev, is_f64, cfg, flags)  # replicated (< 1 % of the time)
    phi, lam, bounds = prepare_problem(img_dev, is_f64, t_dev, a_dev, cfg,
                                       _lambda_mode(flags, cfg), with_bounds=True)
    rank, world = ((dist.get_rank(group), dist.get_world_size(group))
                   if dist.is_initialized() else (0, 1))
    if world == 1:
        # one rank: the whole-image persistent solve (stop rule on the device,
        # no blocks, no host round trips) -- bitwise what dehaze() computes
        from .solver import DeviceProblem, queue_solve_problem

        u, finish = queue_solve_problem(DeviceProblem(phi, lam, h, w, c, c, bounds), cfg,
                                        edge_preserving="no-edge" not in flags)
        out = torch.empty((h, w, c), dtype=torch.float64, device=img_dev.device)
        nat.check(nat.lib().pdz_clamp_interleave(nat.ptr(u), h, w, c, nat.ptr(out), 1,
                                                 nat.stream_ptr()))
        traces = finish()
        return (to_host(out, image),
                DehazeResult(to_host(a_dev, image), to_host(t_dev, image), traces, flags))
    u_slab, traces = solve_slab(phi, lam, h, cfg, edge_preserving="no-edge" not in flags,
                                bounds=bounds, group=group)
    u = _all_gather_rows(u_slab.contiguous(), h, group, rank, world)
    out = torch.empty((h, w, c), dtype=torch.float64, device=img_dev.device)
    nat.check(nat.lib().pdz_clamp_interleave(nat.ptr(u.contiguous()), h, w, c, nat.ptr(out), 1,
                                             nat.stream_ptr()))
    return (to_host(out, image),
            DehazeResult(to_host(a_dev, image), to_host(t_dev, image), traces, flags))
