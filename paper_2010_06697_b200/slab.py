"""Multi-GPU slab decomposition of the projection.

The periodic 3D grid is split along axis 0 into P slabs of n/P planes, one
per rank (one process per GPU).  The local step, the divergence rows, the
FFT along axis 1, the inverse transforms and the gradient pass are local to a
slab apart from one-plane halos; the FFT along axis 0 (with the fused
per-wavevector solve) needs the full axis, which two all-to-all transposes
provide:

  A   T halo exchange (T_c0 = F_c0 - lam_c0/rho on the first / last plane)
      -> stencil divergence + R2C along axis 2            (local)
  B   FFT along axis 1, written straight into the send buffer in
      destination-major order [q][c][i0l][i1l][k2]         (local)
  T1  all-to-all: rank r receives [s][c][i0l][i1l(r)][k2] for every source
      slab s, i.e. all n planes of its n/P-wide block of axis-1 frequencies
  C   FFT along axis 0 + solve + inverse FFT, in place on the receive buffer
  T2  all-to-all back
  D   inverse FFT along axis 1 from the returned send buffer
  E   C2R along axis 2 -> u_tilde                            (local)
  F   u halo exchange -> gradient, multiplier ascent, residual sums

Sums are reduced by all-gathering each rank's fixed-order partials and adding
them in rank order, so results do not depend on the reduction tree.

``exchange="push"`` replaces T1 and T2 by peer-memory stores fused into the
FFT kernels (mm_slab_step FWD_PUSH / SOLVE_PUSH): B writes every output tile
straight into the receive buffer of the rank that owns it, C writes every
solved tile back into its source rank's send buffer, so the transpose
traffic overlaps the transforms tile by tile over NVLink / NVSwitch.  The
peer buffers are mapped once (CUDA IPC handles exchanged through the
communicator; raw pointers when the ranks share a process) and a host
barrier after each step is the only synchronisation -- no kernel waits on
another rank.

``SlabProjector`` is the orchestration; a *backend* supplies the per-rank
compute.  ``DeviceSlabBackend`` calls libmm_admm (CUDA); ``NumpySlabBackend``
restates the same per-rank steps on host arrays with identical buffer
layouts, which lets the orchestration (partitioning, halos, transposes,
global frequency indexing, ordered reductions) be tested on CPU with the
gloo backend (tests/test_slab_gloo.py).
"""

from __future__ import annotations

import numpy as np

__all__ = ["SlabLayout", "SlabProjector", "NumpySlabBackend", "DeviceSlabBackend", "TorchComm",
           "ThreadComm", "SlabSolver"]


class SlabLayout:
    """Geometry of rank `rank`'s slab of an n^3 grid split over `nranks`."""

    def __init__(self, n: int, nranks: int, rank: int, length: float = 0.5, dim: int = 3):
        if dim != 3:
            raise ValueError("slab decomposition is implemented for 3D grids")
        if n % nranks:
            raise ValueError(f"n={n} is not divisible by {nranks} ranks")
        self.n, self.P, self.rank, self.L, self.dim = n, nranks, rank, length, dim
        self.nl = n // nranks
        self.i0 = rank * self.nl          # first global plane
        self.nh = n // 2 + 1
        self.h = 2.0 * length / n

    @property
    def local_shape(self):
        return (self.nl, self.n, self.n)

    @property
    def npts_local(self):
        return self.nl * self.n * self.n

    def plane_slice(self):
        return slice(self.i0, self.i0 + self.nl)

    def neighbours(self):
        return (self.rank - 1) % self.P, (self.rank + 1) % self.P


class TorchComm:
    """Collectives over torch.distributed (NCCL on GPU tensors, gloo on CPU).

    With the gloo backend and device buffers (``cpu_stage``), halo planes
    and partial sums are staged through host memory."""

    def __init__(self, dist, device=None):
        self.dist = dist
        self.device = device
        self.P = dist.get_world_size()
        self.rank = dist.get_rank()
        self.cpu_stage = dist.get_backend() == "gloo"

    def _t(self, a):
        import torch
        t = torch.as_tensor(a)
        if self.cpu_stage:
            return t.cpu()
        return t.to(self.device) if self.device is not None else t

    def barrier(self):
        import torch
        if torch.cuda.is_available():
            torch.cuda.synchronize()
        self.dist.barrier()

    def gather_objects(self, obj):
        out = [None] * self.P
        self.dist.all_gather_object(out, obj)
        return out

    def exchange_halos(self, lo_out, hi_out, lo_in=None, hi_in=None):
        """Send my first plane to the lower neighbour and my last plane to the
        upper one; return (lo_in, hi_in) = (plane below my first, plane above
        my last), received into the given buffers when provided."""
        import torch
        dist = self.dist
        lo_nb, hi_nb = (self.rank - 1) % self.P, (self.rank + 1) % self.P
        lo_out_t, hi_out_t = self._t(lo_out).contiguous(), self._t(hi_out).contiguous()
        lo_in = torch.empty_like(lo_out_t) if lo_in is None else lo_in
        hi_in = torch.empty_like(hi_out_t) if hi_in is None else hi_in
        if self.P == 1:
            lo_in.copy_(hi_out_t)
            hi_in.copy_(lo_out_t)
            return lo_in, hi_in
        lo_rx = torch.empty_like(lo_out_t) if self.cpu_stage else lo_in
        hi_rx = torch.empty_like(hi_out_t) if self.cpu_stage else hi_in
        ops = [dist.P2POp(dist.isend, lo_out_t, lo_nb), dist.P2POp(dist.isend, hi_out_t, hi_nb),
               dist.P2POp(dist.irecv, hi_rx, hi_nb), dist.P2POp(dist.irecv, lo_rx, lo_nb)]
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        if self.cpu_stage:
            lo_in.copy_(lo_rx)
            hi_in.copy_(hi_rx)
        return lo_in, hi_in

    def all_to_all(self, send, out=None):
        """send: tensor/array of shape [P, chunk...]; returns [P, chunk...]."""
        import torch
        s = self._t(send).contiguous()
        out = torch.empty_like(s) if out is None else out
        if self.P == 1:
            out.copy_(s)
            return out
        self.dist.all_to_all_single(out, s)
        return out

    def ordered_sum(self, vec, ops=None):
        """Sum (or max) per slot over ranks in rank order (deterministic)."""
        import torch
        v = torch.as_tensor(np.asarray(vec, dtype=np.float64))
        if self.device is not None and not self.cpu_stage:
            v = v.to(self.device)
        if self.P == 1:
            return np.asarray(vec, dtype=np.float64)
        parts = [torch.empty_like(v) for _ in range(self.P)]
        self.dist.all_gather(parts, v)
        arr = np.stack([p.cpu().numpy() for p in parts])
        out = arr[0].copy()
        for r in range(1, self.P):
            if ops is None:
                out = out + arr[r]
            else:
                out = np.where(np.asarray(ops) == 1, np.maximum(out, arr[r]), out + arr[r])
        return out


def _to_np(x):
    try:
        return x.cpu().numpy()
    except AttributeError:
        return np.asarray(x)


class SlabProjector:
    """Distributed projection + multiplier ascent (solver.py:268-279)."""

    def __init__(self, layout: SlabLayout, backend, comm):
        self.lay = layout
        self.be = backend
        self.comm = comm

    def project_update(self, rho, u_mean):
        """Run stages A-F; returns the global (sum |dG|^2, sum |misfit|^2,
        sum lam (9))."""
        be, comm = self.be, self.comm
        hin = getattr(be, "halo_in", lambda: (None, None))()
        lo, hi = be.boundary_T(rho)                      # A: halos of T_c0
        lo_in, hi_in = comm.exchange_halos(lo, hi, *hin)
        if getattr(be, "push", False):
            be.row_fwd_push(rho, lo_in, hi_in)           # A + B, tiles stored into peers
            comm.barrier()                               # every rank's tiles have landed
            be.col_solve_push()                          # C, tiles stored back into sources
            comm.barrier()
            be.col_inv_from_send(None)                   # D
        else:
            be.row_fwd(rho, lo_in, hi_in)                # A
            send = be.col_fwd_to_send()                  # B
            recv = comm.all_to_all(send, getattr(be, "recv_buffer", lambda: None)())  # T1
            back = be.col_solve(recv)                    # C
            ret = comm.all_to_all(back, getattr(be, "send_buffer", lambda: None)())   # T2
            be.col_inv_from_send(ret)                    # D
        be.row_inv()                                     # E
        ulo, uhi = be.boundary_u()                       # F: halos of u
        ulo_in, uhi_in = comm.exchange_halos(ulo, uhi, *hin)
        local = be.grad_update(rho, u_mean, ulo_in, uhi_in)
        return comm.ordered_sum(local)


class NumpySlabBackend:
    """Host restatement of the per-rank device steps, same buffer layouts.

    Holds F, lam, grad_u (nl, n, n, 3, 3) and u (nl, n, n, 3) of one slab.
    Forward transforms are unnormalised, inverses carry their 1/N, so the
    composite equals the device pipeline's single 1/n^3 in the solve.
    """

    def __init__(self, layout: SlabLayout, F, lam, G, sym_tab, sym_thresh):
        self.lay = layout
        self.F = np.array(F, dtype=float)
        self.lam = np.array(lam, dtype=float)
        self.G = np.array(G, dtype=float)
        self.u = np.zeros(layout.local_shape + (3,))
        self.tab = sym_tab
        self.thresh = sym_thresh

    # -- A ------------------------------------------------------------------
    def boundary_T(self, rho):
        T0 = self.F[..., :, 0] - self.lam[..., :, 0] * (1.0 / rho)   # (nl, n, n, 3)
        return T0[0].copy(), T0[-1].copy()

    def row_fwd(self, rho, lo_in, hi_in):
        lay = self.lay
        T = self.F - self.lam * (1.0 / rho)                         # (nl, n, n, 3, 3)
        T0 = T[..., :, 0]
        T0p = np.concatenate([T0[1:], _to_np(hi_in)[None]], axis=0)  # plane i0+1
        T0m = np.concatenate([_to_np(lo_in)[None], T0[:-1]], axis=0)  # plane i0-1
        d = (T0p - T0m)
        d = d + (np.roll(T[..., :, 1], -1, axis=1) - np.roll(T[..., :, 1], 1, axis=1))
        d = d + (np.roll(T[..., :, 2], -1, axis=2) - np.roll(T[..., :, 2], 1, axis=2))
        self.spec = np.fft.rfft(d, axis=2)                           # (nl, n, nh, 3)
        del lay

    # -- B: FFT along axis 1, destination-major send buffer -------------------
    def col_fwd_to_send(self):
        lay = self.lay
        s = np.fft.fft(self.spec, axis=1)                            # (nl, n, nh, 3)
        P, nl = lay.P, lay.nl
        # [q][c][i0l][i1l][k2]
        send = np.empty((P, 3, nl, nl, lay.nh), dtype=complex)
        for q in range(P):
            send[q] = np.moveaxis(s[:, q * nl:(q + 1) * nl, :, :], -1, 0)
        return send

    # -- C: axis-0 FFT + solve + inverse on the receive buffer ----------------
    def col_solve(self, recv):
        lay = self.lay
        r = _to_np(recv)                                             # [s][c][i0l][i1l][k2]
        P, nl, n = lay.P, lay.nl, lay.n
        full = np.concatenate([r[s] for s in range(P)], axis=1)      # [c][i0][i1l][k2]
        X = np.fft.fft(full, axis=1)
        k1 = lay.rank * nl + np.arange(nl)
        gsq = (self.tab[0][:, None, None] + self.tab[1][k1][None, :, None]) + \
            self.tab[2][: lay.nh][None, None, :]
        inv = np.where(gsq > self.thresh, 1.0 / np.where(gsq > self.thresh, gsq, 1.0), 0.0)
        X = X * (-inv / (2.0 * lay.h))[None]
        x = np.fft.ifft(X, axis=1)
        back = np.stack([x[:, s * nl:(s + 1) * nl] for s in range(P)])
        return back

    # -- D, E ------------------------------------------------------------------
    def col_inv_from_send(self, ret):
        lay = self.lay
        r = _to_np(ret)                                              # [q][c][i0l][i1l][k2]
        s = np.concatenate([np.moveaxis(r[q], 0, -1) for q in range(lay.P)], axis=1)
        self.spec = np.fft.ifft(s, axis=1)

    def row_inv(self):
        self.u = np.fft.irfft(self.spec, n=self.lay.n, axis=2)

    # -- F ------------------------------------------------------------------------
    def boundary_u(self):
        return self.u[0].copy(), self.u[-1].copy()

    def grad_update(self, rho, u_mean, lo_in, hi_in):
        lay = self.lay
        up0 = np.concatenate([self.u[1:], _to_np(hi_in)[None]], axis=0)
        um0 = np.concatenate([_to_np(lo_in)[None], self.u[:-1]], axis=0)
        g = np.empty(lay.local_shape + (3, 3))
        inv2h = 1.0 / (2.0 * lay.h)
        g[..., :, 0] = (up0 - um0) * inv2h
        g[..., :, 1] = (np.roll(self.u, -1, axis=1) - np.roll(self.u, 1, axis=1)) * inv2h
        g[..., :, 2] = (np.roll(self.u, -1, axis=2) - np.roll(self.u, 1, axis=2)) * inv2h
        gnew = g + np.asarray(u_mean).reshape(3, 3)
        dG = gnew - self.G
        mis = gnew - self.F
        self.lam = self.lam + rho * mis
        self.G = gnew
        return np.concatenate([[np.sum(dG * dG), np.sum(mis * mis)],
                               self.lam.reshape(-1, 9).sum(axis=0)])


class ThreadComm:
    """In-process stand-in for TorchComm: P virtual ranks as threads sharing
    one device, exchanging through shared slots and a barrier (used to test
    the device slab path on a single GPU; every kernel runs to completion on
    its own, nothing waits on another rank inside a kernel)."""

    def __init__(self, shared, rank):
        self.sh = shared  # dict: P, barrier, slots
        self.P = shared["P"]
        self.rank = rank

    def _post(self, key, val):
        self.sh["slots"][(key, self.rank)] = val
        self.sh["barrier"].wait()

    def _done(self):
        self.sh["barrier"].wait()

    def exchange_halos(self, lo_out, hi_out, lo_in=None, hi_in=None):
        import torch
        self._post("halo", (lo_out, hi_out))
        lo_nb, hi_nb = (self.rank - 1) % self.P, (self.rank + 1) % self.P
        src_lo = self.sh["slots"][("halo", lo_nb)][1]   # lower neighbour's last plane
        src_hi = self.sh["slots"][("halo", hi_nb)][0]   # upper neighbour's first plane
        lo_in = torch.empty_like(src_lo) if lo_in is None else lo_in
        hi_in = torch.empty_like(src_hi) if hi_in is None else hi_in
        lo_in.copy_(src_lo)
        hi_in.copy_(src_hi)
        torch.cuda.synchronize()
        self._done()
        return lo_in, hi_in

    def all_to_all(self, send, out=None):
        import torch
        self._post("a2a", send)
        out = torch.empty_like(send) if out is None else out
        staged = torch.empty_like(out)
        for s in range(self.P):
            staged[s].copy_(self.sh["slots"][("a2a", s)][self.rank])
        torch.cuda.synchronize()
        self._done()
        out.copy_(staged)
        torch.cuda.synchronize()
        self._done()
        return out

    def barrier(self):
        import torch
        torch.cuda.synchronize()
        self.sh["barrier"].wait()

    def gather_objects(self, obj):
        self._post("obj", obj)
        out = [self.sh["slots"][("obj", r)] for r in range(self.P)]
        self._done()
        return out

    def ordered_sum(self, vec, ops=None):
        self._post("sum", np.asarray(vec, dtype=np.float64).copy())
        arr = [self.sh["slots"][("sum", r)] for r in range(self.P)]
        out = arr[0].copy()
        for r in range(1, self.P):
            if ops is None:
                out = out + arr[r]
            else:
                out = np.where(np.asarray(ops) == 1, np.maximum(out, arr[r]), out + arr[r])
        self._done()
        return out


class DeviceSlabBackend:
    """Per-rank compute through libmm_admm (mm_slab_step); exchange buffers
    are handed to the communicator as zero-copy torch views."""

    def __init__(self, ctx):
        import torch
        from . import _lib
        self.ctx = ctx
        self._lib = _lib

        def view(which, dtype):
            ptr, nbytes = ctx.slab_buffer(which)
            n = nbytes // 8
            arr = _lib.DeviceArray(ptr, (n,), "<f8", owner=ctx)
            t = torch.as_tensor(arr, device=f"cuda:{ctx.device}")
            return t

        P = ctx.slab_P
        self._send = view(_lib.SLAB_BUF_SEND, None).view(P, -1)
        self._recv = view(_lib.SLAB_BUF_RECV, None).view(P, -1)
        self._hol = view(_lib.SLAB_BUF_HALO_OUT_LO, None)
        self._hoh = view(_lib.SLAB_BUF_HALO_OUT_HI, None)
        self._hil = view(_lib.SLAB_BUF_HALO_IN_LO, None)
        self._hih = view(_lib.SLAB_BUF_HALO_IN_HI, None)

    push = False

    def enable_push(self, comm, same_process):
        """Map every rank's RECV and SEND buffers into this context: raw
        device pointers when all ranks live in this process, CUDA IPC
        handles otherwise."""
        lib, ctx = self._lib, self.ctx
        for which in (lib.SLAB_BUF_RECV, lib.SLAB_BUF_SEND):
            if same_process:
                ptrs = comm.gather_objects(ctx.slab_buffer(which)[0])
                ctx.slab_set_peers(which, ptrs)
            else:
                handles = comm.gather_objects(ctx.slab_ipc_handle(which))
                ctx.slab_open_peers(which, handles)
        comm.barrier()
        self.push = True

    def row_fwd_push(self, rho, lo_in, hi_in):
        self._take(self._hil, lo_in)
        self._take(self._hih, hi_in)
        self.ctx.slab_step(self._lib.SLAB_FWD_PUSH, rho)

    def col_solve_push(self):
        self.ctx.slab_step(self._lib.SLAB_SOLVE_PUSH, self._rho)

    def halo_in(self):
        return self._hil, self._hih

    def recv_buffer(self):
        return self._recv

    def send_buffer(self):
        return self._send

    def _take(self, dst, src):
        if src.data_ptr() != dst.data_ptr():
            dst.copy_(src)

    def boundary_T(self, rho):
        self.ctx.slab_step(self._lib.SLAB_HALO_T, rho)
        return self._hol, self._hoh

    def row_fwd(self, rho, lo_in, hi_in):
        self._take(self._hil, lo_in)
        self._take(self._hih, hi_in)
        self.ctx.slab_step(self._lib.SLAB_FWD, rho)

    def col_fwd_to_send(self):
        return self._send

    def col_solve(self, recv):
        self._take(self._recv, recv)
        self.ctx.slab_step(self._lib.SLAB_SOLVE, self._rho)
        return self._recv

    def col_inv_from_send(self, ret):
        if ret is not None:
            self._take(self._send, ret)
        self.ctx.slab_step(self._lib.SLAB_INV, self._rho)

    def row_inv(self):
        pass  # part of SLAB_INV

    def boundary_u(self):
        self.ctx.slab_step(self._lib.SLAB_HALO_U, self._rho)
        return self._hol, self._hoh

    def grad_update(self, rho, u_mean, lo_in, hi_in):
        self._take(self._hil, lo_in)
        self._take(self._hih, hi_in)
        return self.ctx.slab_step(self._lib.SLAB_UPDATE, rho, u_mean)

    def set_rho(self, rho):
        self._rho = rho


class SlabSolver:
    """solve() / outer_iteration() over a slab-decomposed 3D grid (one rank).

    Mirrors solver.py:236-339 with every global quantity (local-step batch
    statistics, means, residual sums) reduced across ranks in rank order, so
    all ranks take identical policy / penalty / convergence decisions.
    Mooney-Rivlin and quadratic materials (pointwise local step); the model
    holds this rank's per-point moduli.
    """

    def __init__(self, layout: SlabLayout, model, bc, params, policy, comm, F, grad_u, lam,
                 rho=None, device=None, exchange="collective"):
        from . import _lib
        from .grid import Grid, axis_symbol_tables
        self.lay, self.model, self.bc, self.params, self.policy, self.comm = (
            layout, model, bc, params, policy, comm)
        n = layout.n
        self.ctx = _lib.Context(3, n=n, length=layout.L, device=device,
                                slab=(layout.P, layout.rank))
        self.ctx.slab_P = layout.P
        tab, thr = axis_symbol_tables(Grid(3, n, layout.L))
        self.ctx.set_symbols(tab, thr)
        model._device_bind(self.ctx, layout.npts_local)
        if hasattr(model, "_phi_scale"):
            # the Armijo noise floor uses the global max mu + max kappa
            mx = comm.ordered_sum([float(np.max(model.mu)), float(np.max(model.kappa))],
                                  ops=[1, 1])
            model._override_max("phi", mx[0] + mx[1])
        self.ctx.upload(_lib.FIELD_F, F)
        self.ctx.upload(_lib.FIELD_G, grad_u)
        self.ctx.upload(_lib.FIELD_LAM, lam)
        self.backend = DeviceSlabBackend(self.ctx)
        if exchange == "push":
            self.backend.enable_push(comm, same_process=isinstance(comm, ThreadComm))
        elif exchange != "collective":
            raise ValueError(f"exchange must be 'collective' or 'push', got {exchange!r}")
        self.proj = SlabProjector(layout, self.backend, comm)
        self.rho = float(params.rho_init if params.rho_init is not None else model.mu_rep)
        if rho is not None:
            self.rho = float(rho)
        self.outer_iter = 0
        self.r_d_prev = np.inf
        self.total_sweeps = 0
        self.history = []
        self.npts = n ** 3
        self.lam_sum = comm.ordered_sum(self.ctx.field_sums(_lib.FIELD_LAM, 9))

    def outer_iteration(self):
        from .materials.base import DeviceLocalStats
        from .projection import macro_gradient
        from .solver import Residuals
        import time
        t0 = time.perf_counter()
        p, pol, model, comm = self.params, self.policy, self.model, self.comm
        npts = self.npts
        tol_pt = pol.target_tol(p, self.r_d_prev)
        sweeps_total = 0
        ops = [0, 0, 1] + [0] * 9
        while True:
            chunk = min(pol.chunk, p.max_local - sweeps_total)
            st = model._device_local(self.ctx, self.lay.npts_local, self.rho, 0.0, chunk, tol_pt)
            g = comm.ordered_sum([st.sum_res2, st.converged_frac * self.lay.npts_local,
                                  st.sweeps] + list(st.sum_F[:9]), ops)
            stats = DeviceLocalStats(None, int(g[2]), g[1] / npts, g[0], g[3:12])
            sweeps_total += stats.sweeps
            if (pol.is_done(stats, sweeps_total) or stats.sweeps < chunk
                    or sweeps_total >= p.max_local):
                break
        self.total_sweeps += sweeps_total
        r_l = float(np.sqrt(stats.sum_res2 / npts)) / model.mu_rep
        F_mean = (np.asarray(stats.sum_F) / npts).reshape(3, 3)
        u_mean = macro_gradient(self.bc, F_mean, (self.lam_sum / npts).reshape(3, 3), self.rho)
        self.backend.set_rho(self.rho)
        sums = self.proj.project_update(self.rho, u_mean)
        self.lam_sum = np.asarray(sums[2:11])
        r_d = self.rho * float(np.sqrt(sums[0] / npts)) / model.mu_rep
        r_p = float(np.sqrt(sums[1] / npts))
        self.u_mean = u_mean
        self.outer_iter += 1
        self.r_d_prev = r_d
        if not np.isfinite(r_p) or r_p > p.divergence_limit:
            from .errors import DivergenceError
            raise DivergenceError(f"primal residual {r_p:.3e} at outer iteration {self.outer_iter}")
        if p.adapt and self.outer_iter > 1:
            rho_ref = p.rho_init if p.rho_init is not None else model.mu_rep
            if r_p > p.tau_adapt * r_d:
                self.rho *= p.kappa_adapt
            elif r_d > p.tau_adapt * r_p:
                self.rho = max(self.rho / p.kappa_adapt, p.rho_min_factor * rho_ref)
        res = Residuals(self.outer_iter, float(r_p), float(r_d), float(r_l), float(self.rho),
                        (time.perf_counter() - t0) * 1e3)
        self.history.append(res)
        return res

    def solve(self, max_outer=None):
        p = self.params
        r_l_tol = p.r_l_tol if p.r_l_tol is not None else max(p.r_p_tol, p.r_d_tol)
        for _ in range(p.max_outer if max_outer is None else max_outer):
            r = self.outer_iteration()
            if r.r_p <= p.r_p_tol and r.r_d <= p.r_d_tol and r.r_l <= r_l_tol:
                return True
        return False

    def fields(self):
        from . import _lib
        sh = self.lay.local_shape
        return {"F": self.ctx.download(_lib.FIELD_F, sh + (3, 3)),
                "grad_u": self.ctx.download(_lib.FIELD_G, sh + (3, 3)),
                "lam": self.ctx.download(_lib.FIELD_LAM, sh + (3, 3)),
                "u_tilde": self.ctx.download(_lib.FIELD_UT, sh + (3,))}
