"""TEST INFRASTRUCTURE: a host (numpy) restatement of one rank's slab
compute -- the per-rank steps of mm_create_slab / mm_slab_step and the
context calls solver.py makes -- with the same buffer layouts the device
backend hands to the communicator (paper_2010_06697_b200/slab.py).  Local
steps call the oracle's C restatement of the reference kernels.

It exists so that the multi-rank orchestration (partitioning, T halos, the
two transposes, global frequency indexing, u and director ghost planes,
rank-ordered reductions, identical decisions on every rank) runs through
the real solve() loop on CPU with torch.distributed gloo
(tests/test_slab_gloo.py).  It is never used by the product package.
"""

from __future__ import annotations

import numpy as np

import oracle
from oracle.core import _p
from paper_2010_06697_b200 import _lib


class _Stats:
    def __init__(self, **kw):
        self.__dict__.update(kw)


def _ls(sum_res2=0.0, n_conv=0, sweeps=0, sum_F=None, sum_nsw=0.0):
    st = _lib.LocalStatsC()
    st.sum_res2 = float(sum_res2)
    st.n_conv = int(n_conv)
    st.sweeps = int(sweeps)
    for i in range(9):
        st.sum_F[i] = 0.0 if sum_F is None or i >= len(sum_F) else float(sum_F[i])
    st.sum_nsw = float(sum_nsw)
    return st


def _us(sum_lam=None):
    us = _lib.UpdateStatsC()
    for i in range(9):
        us.sum_lam[i] = 0.0 if sum_lam is None else float(sum_lam[i])
    return us


class NumpySlabCtx:
    """The _lib.Context calls solver.py / the materials make, on host arrays."""

    NCOMP = {_lib.FIELD_F: 9, _lib.FIELD_G: 9, _lib.FIELD_LAM: 9, _lib.FIELD_UT: 3,
             _lib.FIELD_PREV_F: 9, _lib.FIELD_MOD_A: 1, _lib.FIELD_MOD_B: 1,
             _lib.FIELD_ANG: 2, _lib.FIELD_CHART: 9, _lib.FIELD_PINC: 1, _lib.FIELD_N0: 3,
             _lib.FIELD_FF: 3, _lib.FIELD_PREV_ANG: 2, _lib.FIELD_PREV_CHART: 9,
             _lib.FIELD_PREV_PINC: 1}

    def __init__(self, lay):
        self.lay = lay
        self.n, self.nl = lay.n, lay.nl
        self.npts = lay.npts_local
        self.dim = 3
        self.h = lay.h
        self.f = {}
        nn = lay.n * lay.n
        # u_tilde double buffer with one ghost plane per face: (3, nl + 2, n, n)
        self.ubuf = [np.zeros((3, lay.nl + 2, lay.n, lay.n)) for _ in range(2)]
        self.cur = 0
        self.dirbuf = np.zeros((3, lay.nl + 4, lay.n, lay.n))
        self.ubar = np.zeros(9)
        self.g_implicit = False
        self.lam_pending = False
        self.pending_rho = 0.0
        self.lce = None
        self.res = np.zeros(self.npts)
        self.nsw = np.zeros(self.npts, dtype=np.int64)
        self.ok = np.zeros(self.npts, dtype=bool)
        self.tab = None
        self.thr = None
        del nn

    # -- fields ---------------------------------------------------------------------
    def _u(self, buf=None):
        return self.ubuf[self.cur if buf is None else buf]

    def upload(self, field, arr):
        self._flush()
        a = np.array(arr, dtype=np.float64).reshape(self.npts, -1)
        if field == _lib.FIELD_UT:
            if self.g_implicit:
                self.f[_lib.FIELD_G] = self._gimpl()
                self.g_implicit = False
            u = self._u()
            u[:, 1:self.nl + 1] = a.T.reshape(3, self.nl, self.n, self.n)
            return
        if field == _lib.FIELD_G:
            self.g_implicit = False
        self.f[field] = a

    def add_field(self, field, arr):
        self._flush()
        self.f[field] = self.f[field] + np.asarray(arr, dtype=np.float64).reshape(self.npts, -1)

    def download(self, field, shape):
        self._flush()
        if field == _lib.FIELD_UT:
            u = self._u()[:, 1:self.nl + 1].reshape(3, -1).T
            return np.ascontiguousarray(u).reshape(shape)
        if field == _lib.FIELD_G and self.g_implicit:
            return self._gimpl().reshape(shape)
        return self.f[field].copy().reshape(shape)

    def download_into(self, field, out):
        out[...] = self.download(field, out.shape)
        return out

    def copy_field(self, dst, src):
        self._flush()
        if src == _lib.FIELD_G and self.g_implicit:
            self.f[dst] = self._gimpl()
        else:
            self.f[dst] = self.f[src].copy()

    def field_sums(self, field, ncomp):
        self._flush()
        return self.f[field].sum(axis=0)[:ncomp].copy()

    def set_symbols(self, tab, thr):
        self.tab, self.thr = np.asarray(tab), float(thr)

    def set_option(self, option, value):
        pass

    def set_lce(self, **kw):
        self.lce = dict(kw)

    def synchronize(self):
        pass

    def profile_enable(self, on=True):
        pass

    def profile_read(self, reset=False):
        return ({s: 0.0 for s in _lib.STAGES}, {s: 0 for s in _lib.STAGES})

    def device_bytes(self):
        return 0

    def download_points(self):
        return self.res.copy(), self.nsw.copy(), self.ok.copy()

    # -- stencils on the ghosted u ------------------------------------------------------
    def _grad(self, u, ubar):
        """ubar + central difference of u (3, nl+2, n, n) -> (npts, 9)."""
        nl = self.nl
        inv2h = 1.0 / (2.0 * self.h)
        g = np.empty((nl, self.n, self.n, 3, 3))
        core = u[:, 1:nl + 1]
        for i in range(3):
            g[..., i, 0] = (u[i, 2:nl + 2] - u[i, 0:nl]) * inv2h
            g[..., i, 1] = (np.roll(core[i], -1, axis=1) - np.roll(core[i], 1, axis=1)) * inv2h
            g[..., i, 2] = (np.roll(core[i], -1, axis=2) - np.roll(core[i], 1, axis=2)) * inv2h
        return g.reshape(self.npts, 9) + np.asarray(ubar).reshape(9)

    def _gimpl(self):
        return self._grad(self._u(), self.ubar)

    def _G(self):
        return self._gimpl() if self.g_implicit else self.f[_lib.FIELD_G]

    # -- local step ---------------------------------------------------------------------
    def local_sweeps(self, material, rho, tol, max_sweeps, phi_scale, want_points=False):
        self._flush()
        return self._local(material, rho, tol, max_sweeps, phi_scale)

    def _local(self, material, rho, tol, max_sweeps, phi_scale):
        F = np.ascontiguousarray(self.f[_lib.FIELD_F])
        G = np.ascontiguousarray(self._G())
        L = np.ascontiguousarray(self.f[_lib.FIELD_LAM])
        res = np.empty(self.npts)
        if material == _lib.MAT_LCE:
            return self._lce(F, G, L, rho, tol, max_sweeps)
        mat = 0 if material in (_lib.MAT_MR, _lib.MAT_MR_DESCENT) else 1
        mu = np.ascontiguousarray(self.f[_lib.FIELD_MOD_A].reshape(-1))
        kap = np.ascontiguousarray(self.f.get(_lib.FIELD_MOD_B, self.f[_lib.FIELD_MOD_A])
                                   .reshape(-1))
        sweeps = oracle.lib().orc_descent_sweeps(mat, 3, self.npts, _p(F), _p(G), _p(L), _p(mu),
                                                 _p(kap), float(rho), float(tol),
                                                 int(max_sweeps), float(phi_scale), _p(res))
        self.f[_lib.FIELD_F] = F
        self.res = res
        return _ls(np.sum(res * res), np.sum(res < tol), sweeps, F.sum(axis=0))

    def _lce(self, F, G, L, rho, tol, max_sweeps):
        p = self.lce
        ang = np.ascontiguousarray(self.f[_lib.FIELD_ANG])
        chart = np.ascontiguousarray(self.f[_lib.FIELD_CHART])
        pinc = np.ascontiguousarray(self.f[_lib.FIELD_PINC].reshape(-1))
        n0 = np.ascontiguousarray(self.f[_lib.FIELD_N0])
        ff = np.ascontiguousarray(self.f.get(_lib.FIELD_FF, np.zeros((self.npts, 3))))
        Fk = np.zeros_like(F)
        nk = np.zeros((self.npts, 3))
        res = np.empty(self.npts)
        nsw = np.zeros(self.npts, dtype=np.int64)
        ok = np.zeros(self.npts, dtype=np.uint8)
        oracle.lib().orc_lce3d_sweeps(
            self.npts, _p(F), _p(ang), _p(chart), _p(pinc), _p(G), _p(L), _p(n0), _p(ff),
            _p(Fk), _p(nk), p["mu"], p["r1d"], p["rr"], p["alpha"], p["gamma_inc"], float(rho),
            p["vis_F"], p["vis_n"], float(tol), p["det_tol"], int(max_sweeps), p["phiF_scale"],
            p["phin_scale"], _p(res), _p(nsw), _p(ok))
        self.f[_lib.FIELD_F] = F
        self.f[_lib.FIELD_ANG] = ang
        self.f[_lib.FIELD_CHART] = chart
        self.f[_lib.FIELD_PINC] = pinc.reshape(-1, 1)
        self.res, self.nsw, self.ok = res, nsw, ok.astype(bool)
        return _ls(np.sum(res * res), int(ok.sum()), int(nsw.max()), F.sum(axis=0),
                   float(nsw.sum()))

    # -- the fused ascent ----------------------------------------------------------------
    def _ascend(self):
        G = self._gimpl()
        L = self.f[_lib.FIELD_LAM] + self.pending_rho * (G - self.f[_lib.FIELD_F])
        self.f[_lib.FIELD_LAM] = L
        self.lam_pending = False
        return L.sum(axis=0)

    def _flush(self):
        if self.lam_pending:
            self._ascend()

    def update_multiplier(self):
        return _us(self._ascend())

    def update_and_sweep(self, material, rho_next, tol, max_sweeps, phi_scale, want_points=False):
        lam = self._ascend()
        return self._local(material, rho_next, tol, max_sweeps, phi_scale), _us(lam)


class NumpySlabBackend:
    """Per-rank steps of the slab projection on host arrays (buffer layouts
    of mm_create_slab), torch CPU views for the communicator (gloo)."""

    def __init__(self, lay):
        import torch
        self.lay = lay
        self.ctx = NumpySlabCtx(lay)
        self.device = None
        P, nl, n, nh = lay.P, lay.nl, lay.n, lay.nh
        self._send = np.zeros((P, 3, nl, nl, nh), dtype=np.complex128)
        self._recv = np.zeros_like(self._send)
        self.send = torch.from_numpy(self._send.view(np.float64).reshape(P, -1))
        self.recv = torch.from_numpy(self._recv.view(np.float64).reshape(P, -1))
        self._halo = {k: np.zeros((3, n * n)) for k in ("ol", "oh", "il", "ih")}
        self.halo_out_lo = torch.from_numpy(self._halo["ol"])
        self.halo_out_hi = torch.from_numpy(self._halo["oh"])
        self.halo_in_lo = torch.from_numpy(self._halo["il"])
        self.halo_in_hi = torch.from_numpy(self._halo["ih"])

    def stream(self):
        return 0

    def synchronize(self):
        pass

    def planes(self, which):
        import torch
        c = self.ctx
        if which == _lib.SLAB_FIELD_DIRECTOR:
            arr, g = c.dirbuf, 2
        else:
            arr, g = (c.ubuf[1 - c.cur] if which == _lib.SLAB_FIELD_U_NEW else c._u()), 1
        nl = self.lay.nl

        def plane(comp, z):
            return torch.from_numpy(arr[comp, z + g].reshape(-1))

        tl, tu, fu, fl = [], [], [], []
        for comp in range(3):
            for k in range(g):
                tl.append(plane(comp, k))
                fu.append(plane(comp, nl + k))
                tu.append(plane(comp, nl - g + k))
                fl.append(plane(comp, -g + k))
        return tl, tu, fu, fl

    # -- steps ---------------------------------------------------------------------------
    def step(self, step, rho, u_mean=None):
        c, lay = self.ctx, self.lay
        nl, n = lay.nl, lay.n
        if step == _lib.SLAB_HALO_T:
            c._flush()
            T0 = (c.f[_lib.FIELD_F] - c.f[_lib.FIELD_LAM] * (1.0 / rho)).reshape(
                nl, n, n, 3, 3)[..., :, 0]
            self._halo["ol"][...] = np.moveaxis(T0[0], -1, 0).reshape(3, -1)
            self._halo["oh"][...] = np.moveaxis(T0[-1], -1, 0).reshape(3, -1)
            return None
        if step == _lib.SLAB_FWD:
            T = (c.f[_lib.FIELD_F] - c.f[_lib.FIELD_LAM] * (1.0 / rho)).reshape(nl, n, n, 3, 3)
            lo = self._halo["il"].reshape(3, n, n)
            hi = self._halo["ih"].reshape(3, n, n)
            T0 = np.moveaxis(T[..., :, 0], -1, 0)                        # (3, nl, n, n)
            T0p = np.concatenate([T0[:, 1:], hi[:, None]], axis=1)
            T0m = np.concatenate([lo[:, None], T0[:, :-1]], axis=1)
            T1 = np.moveaxis(T[..., :, 1], -1, 0)
            T2 = np.moveaxis(T[..., :, 2], -1, 0)
            d = (T0p - T0m) + (np.roll(T1, -1, axis=2) - np.roll(T1, 1, axis=2)) + \
                (np.roll(T2, -1, axis=3) - np.roll(T2, 1, axis=3))       # unscaled divergence
            s = np.fft.fft(np.fft.rfft(d, axis=3), axis=2)               # (3, nl, n, nh)
            for q in range(lay.P):
                self._send[q] = s[:, :, q * nl:(q + 1) * nl, :]
            return None
        if step == _lib.SLAB_SOLVE:
            full = np.concatenate([self._recv[s] for s in range(lay.P)], axis=1)  # (3, n, nl, nh)
            X = np.fft.fft(full, axis=1)
            tab = c.tab
            k1 = lay.rank * nl + np.arange(nl)
            gsq = (tab[0][:, None, None] + tab[1][k1][None, :, None]) + \
                tab[2][: lay.nh][None, None, :]
            inv = np.where(gsq > c.thr, 1.0 / np.where(gsq > c.thr, gsq, 1.0), 0.0)
            X = X * (-inv / (2.0 * lay.h))[None]
            x = np.fft.ifft(X, axis=1)
            for s in range(lay.P):
                self._recv[s] = x[:, s * nl:(s + 1) * nl]
            return None
        if step == _lib.SLAB_INV:
            s = np.concatenate([self._send[q] for q in range(lay.P)], axis=2)  # (3, nl, n, nh)
            u = np.fft.irfft(np.fft.ifft(s, axis=2), n=n, axis=3)
            c.ubuf[1 - c.cur][:, 1:nl + 1] = u
            return None
        if step == _lib.SLAB_RES:
            um = np.zeros(9)
            um[: np.size(u_mean)] = np.asarray(u_mean).reshape(-1)
            gold = c._G()
            gnew = c._grad(c.ubuf[1 - c.cur], um)
            dg = gnew - gold
            mis = gnew - c.f[_lib.FIELD_F]
            c.cur = 1 - c.cur
            c.ubar = um
            c.g_implicit = True
            c.lam_pending = True
            c.pending_rho = rho
            out = np.zeros(11)
            out[0], out[1] = np.sum(dg * dg), np.sum(mis * mis)
            return out
        if step == _lib.SLAB_DIRECTOR:
            c._flush()
            ang = c.f[_lib.FIELD_ANG]
            chart = c.f[_lib.FIELD_CHART].reshape(-1, 3, 3)
            ph, th = ang[:, 0], ang[:, 1]
            nloc = np.stack([np.sin(ph) * np.cos(th), np.sin(ph) * np.sin(th), np.cos(ph)], -1)
            nf = np.einsum("pij,pj->pi", chart, nloc)
            c.dirbuf[:, 2:nl + 2] = nf.T.reshape(3, nl, n, n)
            return None
        if step == _lib.SLAB_FRANK:
            p = c.lce
            coef = 2.0 * p["frank_kappa"] / (4.0 * lay.h * lay.h)
            v = c.dirbuf
            core = v[:, 2:nl + 2]
            s = (2.0 * core - v[:, 4:nl + 4]) - v[:, 0:nl]
            s = s + (2.0 * core - np.roll(core, -2, axis=2)) - np.roll(core, 2, axis=2)
            s = s + (2.0 * core - np.roll(core, -2, axis=3)) - np.roll(core, 2, axis=3)
            c.f[_lib.FIELD_FF] = (coef * s).reshape(3, -1).T.copy()
            return None
        raise ValueError(f"step {step} not restated on the host")
