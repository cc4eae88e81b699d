"""Multi-GPU modes of the hot path.

Batch mode (config 3) needs no collective: every rank dehazes its own images
(`dehaze_batch`; `bench.py --gpus N` runs one image per rank).

Row-slab mode (configs 4 and 5, one large image) is implemented here:

* every rank runs the (cheap, < 1 %) front end on the whole image, so all
  ranks hold identical Phi, lambda and tau bounds;
* rank k owns the global rows [y0, y1) = slab_bounds(H, G, k) of ALL C
  planes;
* the solve advances in BLOCKS of k sweeps (temporal blocking): before a
  block the ranks exchange k*R rows with each neighbour (torch.distributed
  point-to-point: NCCL on GPUs, gloo in the CPU tests), R = max(1, K // 2),
  so each rank holds an extended slab of its rows plus up to k*R neighbour
  rows on each side.  One sweep moves information R rows, so after n <= k
  sweeps of the extended slab treated as an image of its own (rows 0 / E-1
  as image borders: exactly the global borders at the top of rank 0 and the
  bottom of rank G-1, fake ones elsewhere) the rank's own rows are exact --
  bit for bit the whole-image arithmetic;
* a block runs on the device as ONE persistent-kernel launch
  (pdz_fixed_point_sweeps_from, include/pdz.h): k sweeps starting from the
  current iterate, counting r^2 only over the rank's own rows;
* the [k][C] table of per-sweep sums of r^2 is all-reduced once per block,
  and every rank applies the same global stop rule (solver.py:347-358) to
  the k sweeps in order; a plane that stopped inside a block takes the
  iterate after its stopping sweep, recomputed from the block's start;
* the final slabs are all-gathered into the full image on every rank.

k trades the redundant halo sweeps (2kR rows per block) against one
exchange + all-reduce + launch per block; the default is
min(4, slab rows // R) (the 2-4 sweeps per launch of the north star;
tools/slab_projection.py measures a rank's block on one GPU).  The block engine is pluggable (`block=`) so the CPU
tests drive the same host logic with an oracle engine on CPU tensors; the
default engine is the CUDA one and there is no CPU fallback in the product.
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


def _cuda_block(cfg: SolverConfig, tau: float, edge_preserving: bool):
    """The product block engine: pdz_fixed_point_sweeps_from on device tensors
    (one persistent launch per block)."""
    import torch

    lib = nat.lib()
    from .solver import _params

    def block(u_ext, phi_e, lam_e, lo, hi, n):
        planes, rows, width = u_ext.shape
        # lambda has one plane shared by all planes: channels = planes
        prm = _params(rows, width, planes, planes, cfg, edge_preserving=edge_preserving,
                      tau=tau, max_iters=n)
        ws = nat.workspace(lib.pdz_solve_workspace_bytes(prm), "slab")
        out = torch.empty_like(u_ext)
        sums = torch.empty((n, planes), dtype=torch.float64, device=u_ext.device)
        failed = torch.empty(planes, dtype=torch.int32, device=u_ext.device)
        nat.check(lib.pdz_fixed_point_sweeps_from(
            prm, nat.ptr(u_ext), nat.ptr(phi_e), nat.ptr(lam_e), int(lo), int(hi), nat.ptr(out),
            nat.ptr(sums), nat.ptr(failed), nat.ptr(ws), ws.numel(), nat.stream_ptr()))
        return out, sums, failed

    return block


def default_sweeps_per_exchange(min_rows: int, halo: int, world: int, max_iters: int) -> int:
    """k of the temporal blocking: one block for a single rank; else at most
    4 sweeps and never deeper than a neighbour's slab (k*R <= its rows)."""
    if world == 1:
        return max(1, max_iters)
    return max(1, min(4, min_rows // halo, max_iters))


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
        k = sweeps_per_exchange or default_sweeps_per_exchange(min_rows, R, world, cfg.max_iters)
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
        self.u = self.phi_e.clone()  # u0 = Phi (solver.py:333)
        self.block = block or _cuda_block(cfg, self.tau, edge_preserving)

    # -- halo exchange -----------------------------------------------------
    def exchange(self, u):
        """Fill the neighbour rows of the extended slab `u` (C, E, W) with the
        neighbours' current rows."""
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
            recv["top"] = torch.empty_like(u[:, :t])
            ops.append(dist.P2POp(dist.irecv, recv["top"], peer, self.group))
        if self.rank < self.world - 1:
            peer = _global_rank(self.group, self.rank + 1)
            b = self.bot
            ops.append(dist.P2POp(dist.isend, u[:, t + n - b:t + n].contiguous(), peer,
                                  self.group))
            recv["bot"] = torch.empty_like(u[:, t + n:])
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
        converged [C])."""
        t, n = self.top, self.rows
        P = self.planes
        u = self.u
        result = u[:, t:t + n].clone()
        running = [True] * P
        prev = [None] * P
        norms = [[] for _ in range(P)]
        iters = [0] * P
        conv = [False] * P
        it = 0
        while it < max_iters and any(running):
            k = min(self.k, max_iters - it)
            self.exchange(u)
            u_new, sums, failed = self.block(u, self.phi_e, self.lam_e, t, t + n, k)
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
                u_s = u_new if s == k else self.block(u, self.phi_e, self.lam_e, t, t + n, s)[0]
                for p, sp in stop_at.items():
                    if sp == s:
                        result[p] = u_s[p, t:t + n]
            u = u_new
            it += k
        self.u = u
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
