"""Multi-GPU slab decomposition of the outer iteration.

The periodic 3D grid is split along axis 0 into P slabs of nl = n/P planes,
one per rank (one process per GPU).  ``solve(..., comm=...)`` runs the same
loop as on one GPU (solver.py's fused schedule, decisions on the host); the
engine then holds a :class:`SlabContext` instead of a single-grid context:
the local step, the fused multiplier-ascent + first-chunk pass and the T
field are slab-local, global quantities (local-step statistics, residual
sums, means) are all-gathered per-rank partials added in rank order (results
independent of the reduction tree, identical decisions on every rank), and
the projection of one iteration is

  HALO_T   T_c0 = (F - lam/rho)_{i,0} of the first / last plane (the fused
           pass's T field)  -> neighbours (one plane each way)
  FWD      stencil divergence + R2C along axis 2, FFT along axis 1, written in
           destination-major order [q][c][i0l][i1l][k2]
  T1       all-to-all (or: FWD_PUSH stores every tile straight into the
           owner's receive buffer over NVLink peer memory, then a barrier)
  SOLVE    FFT along axis 0 + per-wavevector solve + inverse, in place
  T2       all-to-all back (or SOLVE_PUSH peer stores + barrier)
  INV      inverse FFT along axis 1, C2R along axis 2 -> u_new (data planes)
  ghosts   u_new's first / last plane -> the neighbours' ghost planes
  RES      K1: residual sums |dG|^2, |grad_u - F|^2 from the u_new / u_old
           stencils (ghost planes hold the axis-0 neighbours); the ascent
           is left pending for the fused pass

and the LCE frozen data (radius-2 Frank stencil) is DIRECTOR, a two-plane
ghost exchange of the director, FRANK.

Exchanges are issued by a communicator:

* :class:`TorchComm` over ``torch.distributed``.  With NCCL every exchange
  and reduction is issued on the library's CUDA stream
  (``torch.cuda.ExternalStream``), so it is ordered with the kernels around
  it and the host never waits for it (NCCL work on torch's
  current stream was unordered with the library stream); with gloo, device
  buffers are staged through the host after a stream synchronise.
* :class:`ThreadComm`: P virtual ranks as threads of one process sharing one
  GPU (tests); exchanges through shared slots after a stream synchronise.

The per-rank compute is a *backend*: :class:`DeviceSlabBackend` (libmm_admm,
CUDA) here; tests/slab_numpy_backend.py restates it on host arrays with the
oracle's kernels, so the orchestration runs on CPU with gloo.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import ConfigurationError

__all__ = ["SlabLayout", "TorchComm", "ThreadComm", "SlabContext", "DeviceSlabBackend",
           "local_planes", "local_points", "as_comm"]


class SlabLayout:
    """Geometry of rank `rank`'s slab of an n^3 grid split over `nranks`."""

    def __init__(self, n: int, nranks: int, rank: int, length: float = 0.5, dim: int = 3):
        if dim != 3:
            raise ConfigurationError("slab decomposition is implemented for 3D grids")
        if n % nranks:
            raise ConfigurationError(f"n={n} is not divisible by {nranks} ranks")
        if n % 2:
            raise ConfigurationError("slab decomposition needs an even n")
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

    def point_slice(self):
        nn = self.n * self.n
        return slice(self.i0 * nn, (self.i0 + self.nl) * nn)

    def neighbours(self):
        return (self.rank - 1) % self.P, (self.rank + 1) % self.P


def local_planes(grid, comm) -> slice:
    """Axis-0 planes of `grid` this rank holds (index a global field with it)."""
    comm = as_comm(comm)
    return SlabLayout(grid.n, comm.P, comm.rank, grid.length, grid.dim).plane_slice()


def local_points(grid, comm) -> slice:
    """Flattened point range this rank holds (per-point model parameters)."""
    comm = as_comm(comm)
    return SlabLayout(grid.n, comm.P, comm.rank, grid.length, grid.dim).point_slice()


def _combine(arr, ops):
    """Rank-order combination of all-gathered partials: arr (P, k)."""
    out = np.array(arr[0], dtype=np.float64)
    for r in range(1, arr.shape[0]):
        if ops is None:
            out = out + arr[r]
        else:
            out = np.where(np.asarray(ops) == 1, np.maximum(out, arr[r]), out + arr[r])
    return out


# ---------------------------------------------------------------------------
# communicators
# ---------------------------------------------------------------------------

class TorchComm:
    """Exchanges over torch.distributed for one rank.

    exchange="push": the two transposes are the FFT kernels' own NVLink peer
    stores (buffers mapped with CUDA IPC); "collective": NCCL all-to-all."""

    def __init__(self, dist, device=None, exchange="push"):
        if exchange not in ("push", "collective"):
            raise ConfigurationError(f"exchange must be 'push' or 'collective', got {exchange!r}")
        self.dist = dist
        self.device = device
        self.P = dist.get_world_size()
        self.rank = dist.get_rank()
        self.backend = str(dist.get_backend())
        self.exchange = exchange
        self.same_process = False
        self._ext = None
        self._sync = None

    @property
    def stream_ordered(self):
        return self.backend == "nccl"

    def bind(self, stream_ptr, sync, device):
        """Attach the library stream (NCCL work is issued on it) and the
        stream synchronise used before host-side exchanges."""
        self._sync = sync
        self.device = device
        if self.stream_ordered and stream_ptr:
            import torch
            self._ext = torch.cuda.ExternalStream(stream_ptr, device=torch.device("cuda", device))

    def _stream(self):
        import contextlib
        import torch
        if self._ext is not None:
            return torch.cuda.stream(self._ext)
        return contextlib.nullcontext()

    def _host_ready(self, tensors):
        if not self.stream_ordered and any(getattr(t, "is_cuda", False) for t in tensors):
            if self._sync is not None:
                self._sync()

    def _host_done(self, tensors):
        """A host-side exchange wrote device buffers on torch's stream: finish
        it before the library stream reads them."""
        if not self.stream_ordered and any(getattr(t, "is_cuda", False) for t in tensors):
            import torch
            torch.cuda.synchronize(self.device)

    def neighbor_exchange(self, to_lower, to_upper, from_upper, from_lower):
        """to_lower[i] -> the lower neighbour's from_upper[i]; to_upper[i] ->
        the upper neighbour's from_lower[i] (periodic ring of ranks)."""
        import torch
        dist = self.dist
        lo, hi = (self.rank - 1) % self.P, (self.rank + 1) % self.P
        if self.P == 1:
            self._host_ready(list(to_lower) + list(to_upper))
            with self._stream():
                for a, b in zip(to_lower, from_upper):
                    b.copy_(a)
                for a, b in zip(to_upper, from_lower):
                    b.copy_(a)
            self._host_done(list(from_upper) + list(from_lower))
            return
        self._host_ready(list(to_lower) + list(to_upper))
        stage = bool(not self.stream_ordered and to_lower and to_lower[0].is_cuda)
        send_lo = [a.cpu() if stage else a.contiguous() for a in to_lower]
        send_hi = [a.cpu() if stage else a.contiguous() for a in to_upper]
        rx_hi = [torch.empty_like(s) for s in send_lo] if stage else list(from_upper)
        rx_lo = [torch.empty_like(s) for s in send_hi] if stage else list(from_lower)
        ops = []
        for i in range(len(send_lo)):
            ops += [dist.P2POp(dist.isend, send_lo[i], lo), dist.P2POp(dist.isend, send_hi[i], hi),
                    dist.P2POp(dist.irecv, rx_hi[i], hi), dist.P2POp(dist.irecv, rx_lo[i], lo)]
        with self._stream():
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        if stage:
            for a, b in zip(rx_hi, from_upper):
                b.copy_(a)
            for a, b in zip(rx_lo, from_lower):
                b.copy_(a)
            torch.cuda.synchronize(self.device)

    def all_to_all(self, send, recv):
        """send / recv [P, chunk]: block q of send goes to rank q, block s of
        recv comes from rank s."""
        import torch
        if self.P == 1:
            self._host_ready([send])
            with self._stream():
                recv.copy_(send)
            self._host_done([recv])
            return
        self._host_ready([send])
        if not self.stream_ordered and send.is_cuda:
            r = torch.empty_like(send.cpu())
            self.dist.all_to_all_single(r, send.cpu())
            recv.copy_(r)
            torch.cuda.synchronize(self.device)
            return
        with self._stream():
            self.dist.all_to_all_single(recv, send)

    def device_barrier(self):
        """Orders every rank's preceding kernels (peer stores) before the
        next step on any rank: a one-element all-reduce on the library
        stream (NCCL), else stream synchronise + host barrier."""
        import torch
        if self.P == 1:
            return
        if self.stream_ordered:
            with self._stream():
                t = torch.zeros(1, device=torch.device("cuda", self.device))
                self.dist.all_reduce(t)
            return
        if self._sync is not None:
            self._sync()
        self.dist.barrier()

    def barrier(self):
        import torch
        if torch.cuda.is_available():
            torch.cuda.synchronize()
        self.dist.barrier()

    def gather_objects(self, obj):
        out = [None] * self.P
        self.dist.all_gather_object(out, obj)
        return out

    def ordered_sum(self, vec, ops=None):
        """Sum (or max, ops[i] == 1) per slot over ranks in rank order."""
        import torch
        v = np.asarray(vec, dtype=np.float64)
        if self.P == 1:
            return v.copy()
        if self.stream_ordered:
            # every step on the library stream: the upload, the gather and the
            # read-back are ordered with each other and with the library's work
            with self._stream():
                t = torch.as_tensor(v).to(torch.device("cuda", self.device))
                parts = [torch.empty_like(t) for _ in range(self.P)]
                self.dist.all_gather(parts, t)
                arr = np.stack([p.cpu().numpy() for p in parts])
        else:
            t = torch.as_tensor(v)
            parts = [torch.empty_like(t) for _ in range(self.P)]
            self.dist.all_gather(parts, t)
            arr = np.stack([p.numpy() for p in parts])
        return _combine(arr, ops)


class ThreadComm:
    """P virtual ranks as threads sharing one device (tests): exchanges
    through shared slots; a stream synchronise precedes every exchange, so
    no kernel ever waits on another rank."""

    stream_ordered = False
    same_process = True

    def __init__(self, shared, rank, exchange="collective"):
        self.sh = shared  # dict: P, barrier, slots
        self.P = shared["P"]
        self.rank = rank
        self.exchange = exchange
        self._sync = None
        self.device = None

    def bind(self, stream_ptr, sync, device):
        self._sync = sync
        self.device = device

    def _wait(self):
        self.sh["barrier"].wait()

    def _post(self, key, val):
        if self._sync is not None:
            self._sync()
        self.sh["slots"][(key, self.rank)] = val
        self._wait()

    def _finish(self):
        import torch
        if torch.cuda.is_available():
            torch.cuda.synchronize()
        self._wait()

    def neighbor_exchange(self, to_lower, to_upper, from_upper, from_lower):
        self._post("nbx", (list(to_lower), list(to_upper)))
        lo, hi = (self.rank - 1) % self.P, (self.rank + 1) % self.P
        src_hi = self.sh["slots"][("nbx", hi)][0]   # upper neighbour's to_lower
        src_lo = self.sh["slots"][("nbx", lo)][1]   # lower neighbour's to_upper
        staged = [s.clone() for s in src_hi], [s.clone() for s in src_lo]
        self._finish()
        for a, b in zip(staged[0], from_upper):
            b.copy_(a)
        for a, b in zip(staged[1], from_lower):
            b.copy_(a)
        self._finish()

    def all_to_all(self, send, recv):
        self._post("a2a", send)
        staged = [self.sh["slots"][("a2a", s)][self.rank].clone() for s in range(self.P)]
        self._finish()
        for s in range(self.P):
            recv[s].copy_(staged[s])
        self._finish()

    def device_barrier(self):
        if self._sync is not None:
            self._sync()
        self._wait()

    def barrier(self):
        self._finish()

    def gather_objects(self, obj):
        self.sh["slots"][("obj", self.rank)] = obj
        self._wait()
        out = [self.sh["slots"][("obj", r)] for r in range(self.P)]
        self._wait()
        return out

    def ordered_sum(self, vec, ops=None):
        arr = np.stack([np.asarray(v, dtype=np.float64)
                        for v in self.gather_objects(np.asarray(vec, dtype=np.float64).copy())])
        return _combine(arr, ops)


def as_comm(comm):
    """A communicator object, or torch.distributed (default process group)."""
    if comm is None:
        return None
    if hasattr(comm, "neighbor_exchange"):
        return comm
    if hasattr(comm, "get_world_size") and hasattr(comm, "all_to_all_single"):
        import torch
        dev = torch.cuda.current_device() if torch.cuda.is_available() else None
        return TorchComm(comm, dev)
    raise ConfigurationError(f"not a communicator: {comm!r}")


# ---------------------------------------------------------------------------
# per-rank compute: libmm_admm slab context
# ---------------------------------------------------------------------------

class DeviceSlabBackend:
    """One rank's slab on its GPU (mm_create_slab).  Exchange buffers and
    the ghosted fields are handed to the communicator as zero-copy torch
    views."""

    def __init__(self, lay: SlabLayout, device=None):
        import torch
        self.lay = lay
        self.ctx = _lib.Context(3, n=lay.n, length=lay.L, device=device, slab=(lay.P, lay.rank))
        ctx = self.ctx
        self.device = ctx.device
        self._torch = torch
        P = lay.P

        def view(ptr, n):
            arr = _lib.DeviceArray(ptr, (n,), "<f8", owner=ctx)
            return torch.as_tensor(arr, device=torch.device("cuda", ctx.device))

        def buf(which):
            ptr, nbytes = ctx.slab_buffer(which)
            return view(ptr, nbytes // 8)

        self._view = view
        self.send = buf(_lib.SLAB_BUF_SEND).view(P, -1)
        self.recv = buf(_lib.SLAB_BUF_RECV).view(P, -1)
        self.halo_out_lo = buf(_lib.SLAB_BUF_HALO_OUT_LO)
        self.halo_out_hi = buf(_lib.SLAB_BUF_HALO_OUT_HI)
        self.halo_in_lo = buf(_lib.SLAB_BUF_HALO_IN_LO)
        self.halo_in_hi = buf(_lib.SLAB_BUF_HALO_IN_HI)

    def stream(self):
        return self.ctx.slab_stream()

    def synchronize(self):
        self.ctx.synchronize()

    def planes(self, which):
        """Ghost-exchange views of a ghosted field: (to_lower, to_upper,
        from_upper, from_lower) plane lists, one entry per (component, layer)."""
        base, cs, nc, g = self.ctx.slab_field(which)
        lay = self.lay
        nn = lay.n * lay.n
        start = base - 8 * g * nn
        whole = self._view(start, (nc - 1) * cs + (lay.nl + 2 * g) * nn)

        def plane(c, z):   # z in [-g, nl + g)
            o = c * cs + (z + g) * nn
            return whole[o:o + nn]

        tl, tu, fu, fl = [], [], [], []
        for c in range(nc):
            for k in range(g):
                tl.append(plane(c, k))                 # -> lower's plane nl + k
                fu.append(plane(c, lay.nl + k))
                tu.append(plane(c, lay.nl - g + k))    # -> upper's plane -g + k
                fl.append(plane(c, -g + k))
        return tl, tu, fu, fl

    def step(self, step, rho, u_mean=None):
        return self.ctx.slab_step(step, rho, u_mean)

    def enable_push(self, comm):
        """Map every rank's RECV and SEND buffers into this context: raw
        device pointers when all ranks live in this process, CUDA IPC
        handles otherwise."""
        ctx = self.ctx
        for which in (_lib.SLAB_BUF_RECV, _lib.SLAB_BUF_SEND):
            if comm.same_process:
                ptrs = comm.gather_objects(ctx.slab_buffer(which)[0])
                ctx.slab_set_peers(which, ptrs)
            else:
                handles = comm.gather_objects(ctx.slab_ipc_handle(which))
                ctx.slab_open_peers(which, handles)
        comm.barrier()


# ---------------------------------------------------------------------------
# the slab context: the _lib.Context surface the solver uses, distributed
# ---------------------------------------------------------------------------

class SlabContext:
    """Context-like object for one rank's slab (the subset of
    ``_lib.Context`` that solver.py, _engine.py and the materials call).
    Per-point data (fields, moduli, internals) are this rank's slab; every
    returned reduction is global."""

    distributed = True

    def __init__(self, lay: SlabLayout, comm, backend):
        self.lay = lay
        self.comm = comm
        self.be = backend
        self.dim = 3
        self.n = lay.n
        self.npts = lay.npts_local
        self.device = getattr(backend, "device", None)
        self.push = comm.exchange == "push" and lay.P > 1
        comm.bind(backend.stream(), backend.synchronize, self.device)
        if self.push:
            backend.enable_push(comm)

    # -- plumbing passed through to the rank's context ---------------------------
    def __getattr__(self, name):
        # upload / download / download_into / add_field / copy_field /
        # set_symbols / set_option / set_lce / download_points / synchronize /
        # profile_* / device_bytes act on this rank's slab
        return getattr(self.be.ctx, name)

    # -- reductions ---------------------------------------------------------------
    def field_sums(self, field, ncomp):
        return self.comm.ordered_sum(self.be.ctx.field_sums(field, ncomp))

    @staticmethod
    def _local_vec(st):
        return [st.sum_res2, float(st.n_conv), float(st.sweeps)] + list(st.sum_F) + [st.sum_nsw]

    @staticmethod
    def _local_ops():
        return [0, 0, 1] + [0] * 9 + [0]

    @staticmethod
    def _to_local_stats(g):
        st = _lib.LocalStatsC()
        st.sum_res2 = g[0]
        st.n_conv = int(round(g[1]))
        st.sweeps = int(round(g[2]))
        for i in range(9):
            st.sum_F[i] = g[3 + i]
        st.sum_nsw = g[12]
        return st

    def local_sweeps(self, material, rho, tol, max_sweeps, phi_scale, want_points=False):
        if max_sweeps > 64 and material != _lib.MAT_LCE:
            # the descent's 32-sweep stall guard (base.py:224-229) couples all
            # points of the grid; one metered chunk per policy call is <= 64
            raise ConfigurationError(
                "slab decomposition: local chunks above 64 sweeps need the grid-wide stall "
                "guard; use a policy chunk <= 64 (every built-in policy does)")
        st = self.be.ctx.local_sweeps(material, rho, tol, max_sweeps, phi_scale, want_points)
        return self._to_local_stats(self.comm.ordered_sum(self._local_vec(st), self._local_ops()))

    def update_multiplier(self):
        us = self.be.ctx.update_multiplier()
        g = self.comm.ordered_sum(list(us.sum_lam))
        out = _lib.UpdateStatsC()
        for i in range(9):
            out.sum_lam[i] = g[i]
        return out

    def update_and_sweep(self, material, rho_next, tol, max_sweeps, phi_scale, want_points=False):
        ls, us = self.be.ctx.update_and_sweep(material, rho_next, tol, max_sweeps, phi_scale,
                                              want_points)
        g = self.comm.ordered_sum(self._local_vec(ls) + list(us.sum_lam),
                                  self._local_ops() + [0] * 9)
        out = _lib.UpdateStatsC()
        for i in range(9):
            out.sum_lam[i] = g[13 + i]
        return self._to_local_stats(g[:13]), out

    def residuals_and_step(self, prm):
        raise ConfigurationError("slab contexts take the loop's decisions on the host")

    # -- projection ------------------------------------------------------------------
    def project_residuals(self, rho, u_mean):
        """mm_project_residuals over the slabs: returns the global residual
        sums; the ascent is left pending (update_multiplier / update_and_sweep)."""
        be, comm = self.be, self.comm
        be.step(_lib.SLAB_HALO_T, rho)
        comm.neighbor_exchange([be.halo_out_lo], [be.halo_out_hi], [be.halo_in_hi],
                               [be.halo_in_lo])
        if self.push:
            be.step(_lib.SLAB_FWD_PUSH, rho)
            comm.device_barrier()
            be.step(_lib.SLAB_SOLVE_PUSH, rho)
            comm.device_barrier()
        else:
            be.step(_lib.SLAB_FWD, rho)
            comm.all_to_all(be.send, be.recv)
            be.step(_lib.SLAB_SOLVE, rho)
            comm.all_to_all(be.recv, be.send)
        be.step(_lib.SLAB_INV, rho)
        comm.neighbor_exchange(*be.planes(_lib.SLAB_FIELD_U_NEW))
        loc = be.step(_lib.SLAB_RES, rho, u_mean)
        g = comm.ordered_sum(loc[:2])
        out = _lib.UpdateStatsC()
        out.sum_dG2, out.sum_mis2 = float(g[0]), float(g[1])
        return out

    def project_update(self, rho, u_mean):
        """solver.py:268-279 on the slabs: projection, residual sums, ascent."""
        up = self.project_residuals(rho, u_mean)
        lam = self.update_multiplier()
        for i in range(9):
            up.sum_lam[i] = lam.sum_lam[i]
        return up

    def prepare_frozen(self):
        """LCE frozen Frank force (lce.py:223-229): director, two-plane ghost
        exchange, radius-2 stencil."""
        be = self.be
        be.step(_lib.SLAB_DIRECTOR, 1.0)
        self.comm.neighbor_exchange(*be.planes(_lib.SLAB_FIELD_DIRECTOR))
        be.step(_lib.SLAB_FRANK, 1.0)

    def equilibrium_residual(self, material, dt=0.0):
        raise ConfigurationError("equilibrium_residual runs on a single-grid context")

    def project(self, rho, u_mean):
        raise ConfigurationError("helmholtz_project on host arrays runs on a single-grid context")
