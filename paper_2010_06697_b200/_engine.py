"""Device engine: one libmm_admm grid context plus the bookkeeping that keeps
an ADMMState's host views and its device-resident fields consistent.

Ownership model: during solve() the fields live in HBM in SoA
layout; ADMMState attributes materialise read-only host numpy snapshots on
demand (D2H), and assigning a new array marks the field for upload before the
next device operation.
"""

from __future__ import annotations

import os

import numpy as np

from . import _lib
from .grid import Grid, axis_symbol_tables

# ADMMState attribute -> (device field id, rank of the per-point tensor)
STATE_FIELDS = {
    "F": (_lib.FIELD_F, 2),
    "grad_u": (_lib.FIELD_G, 2),
    "lam": (_lib.FIELD_LAM, 2),
    "u_tilde": (_lib.FIELD_UT, 1),
    "prev_F": (_lib.FIELD_PREV_F, 2),
}


class Engine:
    """Device context for one grid (mm_create) with symbols uploaded, or --
    with a communicator -- this rank's slab of it (slab.SlabContext: the
    same surface, global reductions)."""

    def __init__(self, grid: Grid, device=None, comm=None):
        self.grid = grid
        self.comm = comm
        if comm is not None:
            from .slab import DeviceSlabBackend, SlabContext, SlabLayout
            lay = SlabLayout(grid.n, comm.P, comm.rank, grid.length, grid.dim)
            make = getattr(comm, "make_backend", None)
            backend = make(lay) if make is not None else DeviceSlabBackend(lay, device)
            self.ctx = SlabContext(lay, comm, backend)
            self.shape = lay.local_shape
            self.npts = lay.npts_local
        else:
            self.ctx = _lib.Context(grid.dim, n=grid.n, length=grid.length, device=device)
            self.shape = grid.shape
            self.npts = grid.npoints
        tab, thresh = axis_symbol_tables(grid)
        self.ctx.set_symbols(tab, thresh)
        # grad_u storage policy (include/mm_admm.h, MM_OPT_IMPLICIT_GRAD)
        self.ctx.set_option(0, int(os.environ.get("MM_IMPLICIT_GRAD", "0")))
        self.ctx.set_option(1, int(os.environ.get("MM_STENCIL_MARCH", "1")))
        self.ctx.set_option(2, int(os.environ.get("MM_T_FIELD", "1")))
        self.ctx.set_option(3, int(os.environ.get("MM_PLANE_FFT", "1")))
        self.ctx.set_option(4, int(os.environ.get("MM_ROWINV_PIPE", "1")))
        self.ctx.set_option(5, int(os.environ.get("MM_SPECULATE", "1")))
        self.ctx.set_option(6, int(os.environ.get("MM_ROWFWD_WARP", "1")))
        self.ctx.set_option(7, int(os.environ.get("MM_PIPELINE", "1")))
        self.model = None          # model whose parameters are on the device
        self.model_version = None
        self.lam_sum = None        # device-side sum of lam (None: recompute)
        self.point_sweeps = 0.0    # local sweeps summed over points (work counter)

    @property
    def distributed(self) -> bool:
        return self.comm is not None

    def matches(self, grid: Grid, comm=None) -> bool:
        return self.grid == grid and self.comm is comm

    def field_shape(self, rank: int):
        return self.shape + (self.grid.dim,) * rank

    def check_field(self, val, rank, name):
        if self.comm is None:
            self.grid.check_field(val, rank, name)
            return
        want = self.field_shape(rank)
        if np.shape(val) != want:
            from .errors import ConfigurationError
            raise ConfigurationError(f"{name} has shape {np.shape(val)}, this rank's slab is {want}")

    def bind_model(self, model):
        ver = getattr(model, "_device_version", 0)
        if self.model is model and self.model_version == ver:
            return
        model._device_bind(self.ctx, self.npts)
        if self.comm is not None:
            model._globalize(self.comm)
        self.model = model
        self.model_version = ver

    def lam_mean(self):
        d = self.grid.dim
        if self.lam_sum is None:
            self.lam_sum = self.ctx.field_sums(_lib.FIELD_LAM, d * d)
        return (self.lam_sum / self.grid.npoints).reshape(d, d)


def field_shape(grid: Grid, rank: int):
    return grid.shape + (grid.dim,) * rank


_GRID_ENGINES = {}


def scratch_engine(grid: Grid) -> Engine:
    """A cached engine per grid for the stateless helpers (projection,
    stencils) that take host arrays."""
    eng = _GRID_ENGINES.get(grid)
    if eng is None:
        if len(_GRID_ENGINES) > 8:
            _GRID_ENGINES.clear()
        eng = Engine(grid)
        _GRID_ENGINES[grid] = eng
    return eng


def device_discrete_grad(grid: Grid, u: np.ndarray) -> np.ndarray:
    eng = scratch_engine(grid)
    eng.ctx.upload(_lib.FIELD_UT, u)
    eng.ctx.stencil(0)
    return eng.ctx.download(_lib.FIELD_G, field_shape(grid, 2))


def device_discrete_div(grid: Grid, T: np.ndarray) -> np.ndarray:
    eng = scratch_engine(grid)
    eng.ctx.upload(_lib.FIELD_F, T)
    eng.ctx.stencil(1)
    return eng.ctx.download(_lib.FIELD_UT, field_shape(grid, 1))
