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

``SlabProjector`` is the orchestration; a *backend* supplies the per-rank
compute.  ``DeviceSlabBackend`` calls libmm_admm (CUDA); ``NumpySlabBackend``
restates the same per-rank steps on host arrays with identical buffer
layouts, which lets the orchestration (partitioning, halos, transposes,
global frequency indexing, ordered reductions) be tested on CPU with the
gloo backend (tests/test_slab_gloo.py).
"""

from __future__ import annotations

import numpy as np

__all__ = ["SlabLayout", "SlabProjector", "NumpySlabBackend", "TorchComm"]


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
    """Collectives over torch.distributed (NCCL on GPU tensors, gloo on CPU)."""

    def __init__(self, dist, device=None):
        self.dist = dist
        self.device = device
        self.P = dist.get_world_size()
        self.rank = dist.get_rank()

    def _t(self, a):
        import torch
        t = torch.as_tensor(a)
        return t.to(self.device) if self.device is not None else t

    def exchange_halos(self, lo_out, hi_out):
        """Send my first plane to the lower neighbour and my last plane to the
        upper one; return (lo_in, hi_in) = (plane below my first, plane above
        my last)."""
        import torch
        dist = self.dist
        lo_nb, hi_nb = (self.rank - 1) % self.P, (self.rank + 1) % self.P
        lo_out_t, hi_out_t = self._t(lo_out).contiguous(), self._t(hi_out).contiguous()
        lo_in = torch.empty_like(lo_out_t)
        hi_in = torch.empty_like(hi_out_t)
        if self.P == 1:
            return hi_out_t, lo_out_t
        ops = [dist.P2POp(dist.isend, lo_out_t, lo_nb), dist.P2POp(dist.isend, hi_out_t, hi_nb),
               dist.P2POp(dist.irecv, hi_in, hi_nb), dist.P2POp(dist.irecv, lo_in, lo_nb)]
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        return lo_in, hi_in

    def all_to_all(self, send):
        """send: tensor/array of shape [P, chunk...]; returns [P, chunk...]."""
        import torch
        s = self._t(send).contiguous()
        out = torch.empty_like(s)
        if self.P == 1:
            out.copy_(s)
            return out
        self.dist.all_to_all_single(out, s)
        return out

    def ordered_sum(self, vec, ops=None):
        """Sum (or max) per slot over ranks in rank order (deterministic)."""
        import torch
        v = torch.as_tensor(np.asarray(vec, dtype=np.float64))
        if self.device is not None:
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
        lo, hi = be.boundary_T(rho)                      # A: halos of T_c0
        lo_in, hi_in = comm.exchange_halos(lo, hi)
        be.row_fwd(rho, lo_in, hi_in)                    # A
        send = be.col_fwd_to_send()                      # B
        recv = comm.all_to_all(send)                     # T1
        back = be.col_solve(recv)                        # C
        ret = comm.all_to_all(back)                      # T2
        be.col_inv_from_send(ret)                        # D
        be.row_inv()                                     # E
        ulo, uhi = be.boundary_u()                       # F: halos of u
        ulo_in, uhi_in = comm.exchange_halos(ulo, uhi)
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
