"""Multi-GPU modes of the hot path.

Batch mode (config 3) needs no collective: every rank dehazes its own images
(`dehaze_batch`; `bench.py --gpus N` runs one image per rank).

Row-slab mode (configs 4 and 5, one large image) is implemented here:

* every rank runs the (cheap, < 1 %) front end on the whole image, so all
  ranks hold identical Phi, lambda and tau bounds;
* rank k owns the global rows [y0, y1) = slab_bounds(H, G, k) of ALL C
  planes, stored as an extended slab of R + (y1 - y0) + R rows,
  R = max(1, K // 2);
* before every sweep the R halo rows are exchanged with the neighbouring
  ranks (torch.distributed point-to-point: NCCL on GPUs, gloo in the CPU
  tests); at the global top / bottom the halo is the symmetric reflection of
  the slab's own rows (np.pad "symmetric", solver.py:235);
* one sweep of the slab runs on the device through
  pdz_fixed_point_step_rows (include/pdz.h), which knows the global row of
  every array row -- np.gradient's one-sided rows (solver.py:178-179) exist
  only at the global border, and the reflected halo makes the zero-flux
  border (solver.py:205-209) exact;
* the per-plane sums of r^2 are all-reduced every sweep, so every rank
  applies the same global stop rule (solver.py:347-358);
* the final slabs are all-gathered into the full image on every rank.

The sweep itself is pluggable (`step=`) so the CPU tests can drive the same
host logic with an oracle step on CPU tensors; the default step is the CUDA
one and there is no CPU fallback in the product.
"""

from __future__ import annotations

import logging
import math

from . import _native as nat
from .config import DehazeResult, SolverConfig, SolverTrace, normalize_ablation
from .image import to_host, validate_image

logger = logging.getLogger("pdehaze.solver")

__all__ = ["slab_bounds", "halo_rows", "SlabSolver", "solve_slab", "dehaze_slabs"]


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


def _cuda_step(cfg: SolverConfig, tau: float, edge_preserving: bool):
    """The product sweep: pdz_fixed_point_step_rows on device tensors."""
    import torch

    lib = nat.lib()
    from .solver import _params

    def step(u_in, u_out, phi_e, lam_e, y_off, height, row_lo, row_hi):
        planes, rows, width = u_in.shape
        prm = _params(rows, width, planes, planes, cfg, edge_preserving=edge_preserving, tau=tau)
        ws = nat.workspace(lib.pdz_step_workspace_bytes(prm), "slab")
        sums = torch.empty(planes, dtype=torch.float64, device=u_in.device)
        nf = torch.empty(planes, dtype=torch.int32, device=u_in.device)
        nat.check(lib.pdz_fixed_point_step_rows(
            prm, nat.ptr(u_in), nat.ptr(u_out), nat.ptr(phi_e), nat.ptr(lam_e), int(y_off),
            int(height), int(row_lo), int(row_hi), nat.ptr(sums), nat.ptr(nf), nat.ptr(ws),
            ws.numel(), nat.stream_ptr()))
        return sums, nf

    return step


class SlabSolver:
    """One rank's share of a row-slab solve.

    phi: (C, H, W) full Phi (every rank holds it after the replicated front
    end) or just this rank's rows (C, y1 - y0, W) with `full=False`;
    lam: (H, W) or (y1 - y0, W) likewise.
    """

    def __init__(self, phi, lam, height: int, cfg: SolverConfig, *, tau: float,
                 edge_preserving: bool = True, group=None, rank: int = 0, world: int = 1,
                 full: bool = True, step=None):
        import torch

        self.cfg, self.tau, self.height = cfg, float(tau), int(height)
        self.group, self.rank, self.world = group, rank, world
        self.y0, self.y1 = slab_bounds(self.height, world, rank)
        self.rows = self.y1 - self.y0
        self.halo = R = halo_rows(cfg.kernel_size)
        last_rows = self.height - slab_bounds(self.height, world, world - 1)[0]
        if last_rows < R or self.rows < R:
            raise ValueError(f"{world} row slabs of a {self.height}-row image leave fewer than "
                             f"the {R} halo rows per slab")
        planes, _, width = phi.shape
        self.planes, self.width = planes, width
        E = self.rows + 2 * R
        kw = dict(dtype=phi.dtype, device=phi.device)
        self.phi_e = torch.zeros((planes, E, width), **kw)
        self.lam_e = torch.zeros((E, width), dtype=lam.dtype, device=lam.device)
        src_phi = phi[:, self.y0:self.y1] if full else phi
        src_lam = lam[self.y0:self.y1] if full else lam
        self.phi_e[:, R:R + self.rows] = src_phi
        self.lam_e[R:R + self.rows] = src_lam
        self.u = [self.phi_e.clone(), torch.zeros_like(self.phi_e)]  # u0 = Phi (solver.py:333)
        self.step = step or _cuda_step(cfg, self.tau, edge_preserving)
        self._recv = [torch.empty((planes, R, width), **kw) for _ in range(2)]

    # -- halo exchange -----------------------------------------------------
    def exchange(self, u):
        """Fill the R halo rows above and below the slab of `u` (C, E, W)."""
        import torch

        R, n = self.halo, self.rows
        ops = []
        if self.world > 1:
            import torch.distributed as dist

            if self.rank > 0:
                peer = _global_rank(self.group, self.rank - 1)
                ops.append(dist.P2POp(dist.isend, u[:, R:2 * R].contiguous(), peer, self.group))
                ops.append(dist.P2POp(dist.irecv, self._recv[0], peer, self.group))
            if self.rank < self.world - 1:
                peer = _global_rank(self.group, self.rank + 1)
                ops.append(dist.P2POp(dist.isend, u[:, n:n + R].contiguous(), peer, self.group))
                ops.append(dist.P2POp(dist.irecv, self._recv[1], peer, self.group))
            for req in dist.batch_isend_irecv(ops) if ops else []:
                req.wait()
        if self.rank > 0:
            u[:, :R] = self._recv[0]
        else:  # global top: rows -1-i <- i
            u[:, :R] = torch.flip(u[:, R:2 * R], dims=[1])
        if self.rank < self.world - 1:
            u[:, n + R:] = self._recv[1]
        else:  # global bottom: rows H+i <- H-1-i
            u[:, n + R:] = torch.flip(u[:, n:n + R], dims=[1])

    def _allreduce(self, sums, nf):
        if self.world > 1:
            import torch.distributed as dist

            dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=self.group)
            dist.all_reduce(nf, op=dist.ReduceOp.MAX, group=self.group)
        return sums, nf

    # -- the solve -----------------------------------------------------------
    def solve(self, max_iters: int, rel_tol: float):
        """fixed_point_solve (solver.py:343-358) of every plane over the slab.
        Returns (u slab (C, y1 - y0, W), norms [C] lists, iterations [C],
        converged [C])."""
        R, n = self.halo, self.rows
        P = self.planes
        result = self.u[0][:, R:R + n].clone()
        running = [True] * P
        prev = [None] * P
        norms = [[] for _ in range(P)]
        iters = [0] * P
        conv = [False] * P
        cur = 0
        for it in range(1, max_iters + 1):
            u_in, u_out = self.u[cur], self.u[cur ^ 1]
            self.exchange(u_in)
            sums, nf = self.step(u_in, u_out, self.phi_e, self.lam_e, self.y0 - R, self.height,
                                 R, R + n)
            sums, nf = self._allreduce(sums, nf)
            sums_h = sums.to("cpu").numpy()
            nf_h = nf.to("cpu").numpy()
            cur ^= 1
            for p in range(P):
                if not running[p]:
                    continue
                if nf_h[p]:
                    raise FloatingPointError(
                        f"solver produced non-finite values at iteration {it}")
                nrm = math.sqrt(float(sums_h[p]))
                norms[p].append(nrm)
                iters[p] = it
                stop = False
                if prev[p] is not None and abs(nrm - prev[p]) / max(prev[p], 1e-30) <= rel_tol:
                    conv[p] = stop = True
                elif it >= max_iters:
                    stop = True
                prev[p] = nrm
                if stop:  # the answer is the iterate after the stopping update
                    running[p] = False
                    result[p] = self.u[cur][p, R:R + n]
            if not any(running):
                break
        return result, norms, iters, conv


def solve_slab(phi, lam, height, cfg: SolverConfig, *, tau=None, edge_preserving=True,
               bounds=None, group=None, step=None, full=True, warn=True):
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
                        group=group, rank=rank, world=world, full=full, step=step)
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
    u_slab, traces = solve_slab(phi, lam, h, cfg, edge_preserving="no-edge" not in flags,
                                bounds=bounds, group=group)
    u = _all_gather_rows(u_slab.contiguous(), h, group, rank, world)
    out = torch.empty((h, w, c), dtype=torch.float64, device=img_dev.device)
    nat.check(nat.lib().pdz_clamp_interleave(nat.ptr(u.contiguous()), h, w, c, nat.ptr(out), 1,
                                             nat.stream_ptr()))
    return (to_host(out, image),
            DehazeResult(to_host(a_dev, image), to_host(t_dev, image), traces, flags))
