"""ctypes binding of libmm_admm.so (include/mm_admm.h) and the device
context wrapper used by the host package.

There is no CPU fallback: if the extension is missing or no CUDA device is
visible, every call that needs the device raises RuntimeError.
"""

from __future__ import annotations

import ctypes
import mmap
import os
import threading

import numpy as np

from .errors import (
    ConfigurationError,
    DivergenceError,
    InadmissibleStateError,
    ParameterError,
)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libmm_admm.so")

MM_OK, MM_ERR_PARAM, MM_ERR_CONFIG, MM_ERR_INADMISSIBLE, MM_ERR_DIVERGED, MM_ERR_CUDA = range(6)

FIELD_F, FIELD_G, FIELD_LAM, FIELD_UT, FIELD_PREV_F, FIELD_MOD_A, FIELD_MOD_B = range(7)
FIELD_ANG, FIELD_CHART, FIELD_PINC, FIELD_N0, FIELD_FF, FIELD_PREV_ANG, FIELD_PREV_CHART = range(7, 14)
FIELD_PREV_PINC = 14

MAT_MR, MAT_QUADRATIC, MAT_LCE, MAT_MR_DESCENT = range(4)
POLICY_EXACT, POLICY_FRACTION, POLICY_RATIO = range(3)

# every symbol include/mm_admm.h declares (checked by the CPU test suite)
EXPORTS = (
    "mm_abi_version", "mm_struct_size", "mm_create", "mm_create_points", "mm_destroy", "mm_last_error",
    "mm_synchronize", "mm_device_bytes", "mm_upload", "mm_download", "mm_copy_field",
    "mm_field_sums", "mm_set_symbols", "mm_local_sweeps", "mm_set_lce", "mm_download_points",
    "mm_prepare_frozen", "mm_project", "mm_project_update", "mm_stencil",
    "mm_profile_enable", "mm_profile_read", "mm_frank_stencil", "mm_set_option",
    "mm_project_residuals", "mm_update_multiplier", "mm_update_and_sweep",
    "mm_create_slab", "mm_slab_buffer", "mm_slab_step", "mm_add_field",
    "mm_equilibrium_residual", "mm_selftest_log", "mm_slab_set_peers", "mm_slab_ipc_handle",
    "mm_slab_open_peers", "mm_bloch_setup", "mm_bloch_start", "mm_bloch_iterate",
    "mm_bloch_mode", "mm_debug_lce_counters", "mm_residuals_and_step", "mm_slab_field",
    "mm_slab_stream", "mm_solve_fused",
)

SLAB_HALO_T, SLAB_FWD, SLAB_SOLVE, SLAB_INV = range(4)
SLAB_FWD_PUSH, SLAB_SOLVE_PUSH, SLAB_RES, SLAB_DIRECTOR, SLAB_FRANK = 7, 8, 9, 10, 11
SLAB_FIELD_U_NEW, SLAB_FIELD_U, SLAB_FIELD_DIRECTOR = range(3)
SLAB_BUF_SEND, SLAB_BUF_RECV, SLAB_BUF_HALO_OUT_LO, SLAB_BUF_HALO_OUT_HI = range(4)
SLAB_BUF_HALO_IN_LO, SLAB_BUF_HALO_IN_HI = 4, 5

STAGES = ("local", "row_fwd", "col_fwd", "col_solve", "col_inv", "row_inv", "grad", "frozen",
          "other", "fused", "plane")


class LocalStatsC(ctypes.Structure):
    _fields_ = [("sweeps", ctypes.c_int64), ("n_conv", ctypes.c_int64),
                ("sum_res2", ctypes.c_double), ("sum_F", ctypes.c_double * 9),
                ("sum_nsw", ctypes.c_double)]


class UpdateStatsC(ctypes.Structure):
    _fields_ = [("sum_dG2", ctypes.c_double), ("sum_mis2", ctypes.c_double),
                ("sum_lam", ctypes.c_double * 9)]


class StepParamsC(ctypes.Structure):
    _fields_ = [("u_mean", ctypes.c_double * 9), ("rho", ctypes.c_double),
                ("npts", ctypes.c_double), ("mu_rep", ctypes.c_double), ("r_l", ctypes.c_double),
                ("r_p_tol", ctypes.c_double), ("r_d_tol", ctypes.c_double),
                ("r_l_tol", ctypes.c_double), ("divergence_limit", ctypes.c_double),
                ("adapt", ctypes.c_int), ("tau_adapt", ctypes.c_double),
                ("kappa_adapt", ctypes.c_double), ("rho_floor", ctypes.c_double),
                ("outer_iter", ctypes.c_int64), ("last_allowed", ctypes.c_int),
                ("ratio_policy", ctypes.c_int), ("point_tol", ctypes.c_double),
                ("ratio", ctypes.c_double), ("material", ctypes.c_int),
                ("phi_scale", ctypes.c_double), ("chunk", ctypes.c_int64)]


class StepResultC(ctypes.Structure):
    _fields_ = [("r_p", ctypes.c_double), ("r_d", ctypes.c_double), ("rho_next", ctypes.c_double),
                ("diverged", ctypes.c_int), ("done", ctypes.c_int), ("swept", ctypes.c_int),
                ("sum_lam", ctypes.c_double * 9)]


class SolveParamsC(ctypes.Structure):
    _fields_ = [("step", StepParamsC), ("bc_mask", ctypes.c_double * 9),
                ("bc_value", ctypes.c_double * 9), ("rho", ctypes.c_double),
                ("r_d_prev", ctypes.c_double), ("lam_sum", ctypes.c_double * 9),
                ("outer_iter", ctypes.c_int64), ("max_outer", ctypes.c_int64),
                ("max_local", ctypes.c_int64), ("policy", ctypes.c_int),
                ("policy_chunk", ctypes.c_int64), ("fraction", ctypes.c_double)]


class SolveResultC(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int64), ("outer_iter", ctypes.c_int64),
                ("total_sweeps", ctypes.c_int64), ("converged", ctypes.c_int),
                ("diverged", ctypes.c_int), ("rho", ctypes.c_double),
                ("r_d_prev", ctypes.c_double), ("point_sweeps", ctypes.c_double),
                ("lam_sum", ctypes.c_double * 9), ("u_mean", ctypes.c_double * 9)]


class ProfileC(ctypes.Structure):
    _fields_ = [("ms", ctypes.c_double * 11), ("launches", ctypes.c_int64 * 11)]


class LCEParamsC(ctypes.Structure):
    _fields_ = [(name, ctypes.c_double) for name in
                ("mu", "r1d", "rr", "alpha", "gamma_inc", "vis_F", "vis_n", "det_tol",
                 "phiF_scale", "phin_scale", "frank_kappa")]


_lib = None
_lock = threading.Lock()

_HUGE_MIN_BYTES = 64 << 20


_prefaulted = {}   # (shape, dtype) -> a touched host array ready for a download
_prefault_lock = threading.Lock()


def prefault_async(shapes, dtype=np.float64, threads=4):
    """Allocate and touch host arrays for downloads expected after the
    device work now in flight (solve() calls it for fields the caller had on
    the host): first-touch page faults, the slow part of a download into
    fresh memory (27 vs 55 GB/s), then overlap the GPU iterations.  One
    array per shape is kept; host_empty() hands it out."""
    dt = np.dtype(dtype)

    def work(shape):
        a = _host_empty_raw(shape, dt)
        nb = a.nbytes
        step = max(1, (nb + threads - 1) // threads)
        base = a.ctypes.data
        ts = [threading.Thread(target=ctypes.memset, args=(base + o, 0, min(step, nb - o)))
              for o in range(0, nb, step)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        with _prefault_lock:
            _prefaulted[(tuple(shape), dt.str)] = a

    for shape in shapes:
        key = (tuple(shape), dt.str)
        with _prefault_lock:
            _prefaulted.pop(key, None)
        if int(np.prod(shape)) * dt.itemsize >= _HUGE_MIN_BYTES:
            threading.Thread(target=work, args=(tuple(shape),), daemon=True).start()


def host_empty(shape, dtype=np.float64):
    """Host array for a field download: a pre-faulted one when prefault_async
    prepared it, else a fresh one (see _host_empty_raw)."""
    dt = np.dtype(dtype)
    with _prefault_lock:
        a = _prefaulted.pop((tuple(shape), dt.str), None)
    if a is not None:
        return a
    return _host_empty_raw(shape, dt)


def _host_empty_raw(shape, dtype=np.float64):
    """Large host arrays are backed by an anonymous mapping advised for
    transparent huge pages: the first write into fresh memory (the library's
    multi-threaded copy out of its pinned stage) then faults in 2 MiB pages
    instead of 4 KiB ones (~1.5x faster on the B200 hosts)."""
    dt = np.dtype(dtype)
    nbytes = int(np.prod(shape)) * dt.itemsize
    if nbytes < _HUGE_MIN_BYTES or not hasattr(mmap, "MADV_HUGEPAGE"):
        return np.empty(shape, dtype=dt)
    m = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    try:
        m.madvise(mmap.MADV_HUGEPAGE)
    except OSError:
        pass
    return np.frombuffer(m, dtype=dt).reshape(shape)


def load_library():
    """Load the CUDA extension (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"CUDA extension not built: {LIB_PATH} is missing "
                "(run `python -m paper_2010_06697_b200.build`); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        P, D, I64, I = ctypes.c_void_p, ctypes.c_double, ctypes.c_int64, ctypes.c_int
        PP = ctypes.POINTER(ctypes.c_void_p)
        sig = {
            "mm_abi_version": ([], I),
            "mm_struct_size": ([I], I64),
            "mm_create": ([I, I, D, I, PP], I),
            "mm_create_points": ([I, I64, I, PP], I),
            "mm_destroy": ([P], None),
            "mm_last_error": ([P], ctypes.c_char_p),
            "mm_synchronize": ([P], I),
            "mm_device_bytes": ([P], I64),
            "mm_upload": ([P, I, P, I64], I),
            "mm_download": ([P, I, P, I64], I),
            "mm_copy_field": ([P, I, I], I),
            "mm_field_sums": ([P, I, P], I),
            "mm_set_symbols": ([P, P, D], I),
            "mm_local_sweeps": ([P, I, D, D, I64, D, I, ctypes.POINTER(LocalStatsC)], I),
            "mm_set_lce": ([P, ctypes.POINTER(LCEParamsC)], I),
            "mm_download_points": ([P, P, P, P, I64], I),
            "mm_prepare_frozen": ([P], I),
            "mm_project": ([P, D, P], I),
            "mm_project_update": ([P, D, P, ctypes.POINTER(UpdateStatsC)], I),
            "mm_stencil": ([P, I], I),
            "mm_profile_enable": ([P, I], I),
            "mm_frank_stencil": ([P], I),
            "mm_set_option": ([P, I, I64], I),
            "mm_project_residuals": ([P, D, P, ctypes.POINTER(UpdateStatsC)], I),
            "mm_create_slab": ([I, D, I, I, I, PP], I),
            "mm_slab_buffer": ([P, I, PP, ctypes.POINTER(I64)], I),
            "mm_slab_step": ([P, I, D, P, P], I),
            "mm_update_multiplier": ([P, ctypes.POINTER(UpdateStatsC)], I),
            "mm_update_and_sweep": ([P, I, D, D, I64, D, I, ctypes.POINTER(LocalStatsC),
                                     ctypes.POINTER(UpdateStatsC)], I),
            "mm_profile_read": ([P, ctypes.POINTER(ProfileC), I], I),
            "mm_add_field": ([P, I, P, I64], I),
            "mm_equilibrium_residual": ([P, I, D, ctypes.POINTER(D)], I),
            "mm_selftest_log": ([P, P, P, I64], I),
            "mm_slab_set_peers": ([P, I, P, I], I),
            "mm_slab_ipc_handle": ([P, I, P], I),
            "mm_slab_open_peers": ([P, I, P, I], I),
            "mm_bloch_setup": ([P, P, P, P, P, P, D, D], I),
            "mm_bloch_start": ([P, P], I),
            "mm_bloch_iterate": ([P, I, D, D, D, D, P], I),
            "mm_bloch_mode": ([P, P], I),
            "mm_debug_lce_counters": ([P, I], I),
            "mm_slab_field": ([P, I, PP, ctypes.POINTER(I64), ctypes.POINTER(I),
                               ctypes.POINTER(I)], I),
            "mm_slab_stream": ([P, PP], I),
            "mm_solve_fused": ([P, ctypes.POINTER(SolveParamsC), ctypes.POINTER(SolveResultC),
                                P], I),
            "mm_residuals_and_step": ([P, ctypes.POINTER(StepParamsC), ctypes.POINTER(StepResultC),
                                       ctypes.POINTER(LocalStatsC)], I),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
        return L


_EXC = {
    MM_ERR_PARAM: ParameterError,
    MM_ERR_CONFIG: ConfigurationError,
    MM_ERR_INADMISSIBLE: InadmissibleStateError,
    MM_ERR_DIVERGED: DivergenceError,
}


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data)


def _require_device(device):
    import torch  # noqa: PLC0415  (plumbing only: device discovery)
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device visible: the B200 path has no CPU fallback")
    return int(device if device is not None else torch.cuda.current_device())


class Context:
    """One device context (mm_ctx): a periodic grid, or a bare point set."""

    def __init__(self, dim, n=None, length=None, npts=None, device=None, slab=None):
        self.lib = load_library()
        self.device = _require_device(device)
        self.dim = int(dim)
        h = ctypes.c_void_p()
        if slab is not None:
            nranks, rank = slab
            rc = self.lib.mm_create_slab(int(n), float(length), int(nranks), int(rank),
                                         self.device, ctypes.byref(h))
            self.npts = (int(n) // int(nranks)) * int(n) ** 2
            self.n = int(n)
        elif n is not None:
            rc = self.lib.mm_create(self.dim, int(n), float(length), self.device, ctypes.byref(h))
            self.npts = int(n) ** self.dim
            self.n = int(n)
        else:
            rc = self.lib.mm_create_points(self.dim, int(npts), self.device, ctypes.byref(h))
            self.npts = int(npts)
            self.n = None
        self.h = h
        if rc != MM_OK:
            msg = self.lib.mm_last_error(h).decode() if h.value else "context creation failed"
            if h.value:
                self.lib.mm_destroy(h)
            self.h = None
            self._raise(rc, msg)

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value and _lib is not None:
            try:
                _lib.mm_destroy(h)
            except Exception:
                pass
            self.h = None

    def close(self):
        self.__del__()

    @staticmethod
    def _raise(rc, msg):
        exc = _EXC.get(rc)
        if exc is None:
            raise RuntimeError(f"libmm_admm: {msg}")
        raise exc(msg)

    def check(self, rc):
        if rc != MM_OK:
            self._raise(rc, self.lib.mm_last_error(self.h).decode())

    # -- transfers -------------------------------------------------------
    def upload(self, field, arr):
        a = np.ascontiguousarray(arr, dtype=np.float64)
        self.check(self.lib.mm_upload(self.h, field, _ptr(a), a.size))

    def add_field(self, field, arr):
        """field += arr on the device (one rounding per element)."""
        a = np.ascontiguousarray(arr, dtype=np.float64)
        self.check(self.lib.mm_add_field(self.h, field, _ptr(a), a.size))

    def equilibrium_residual(self, material, dt=0.0):
        out = ctypes.c_double()
        self.check(self.lib.mm_equilibrium_residual(self.h, int(material), float(dt),
                                                    ctypes.byref(out)))
        return out.value

    def selftest_log(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty_like(x)
        self.check(self.lib.mm_selftest_log(self.h, _ptr(x), _ptr(y), x.size))
        return y

    def download(self, field, shape):
        out = host_empty(shape)
        self.check(self.lib.mm_download(self.h, field, _ptr(out), out.size))
        return out

    def download_into(self, field, out):
        assert out.flags.c_contiguous and out.dtype == np.float64
        self.check(self.lib.mm_download(self.h, field, _ptr(out), out.size))
        return out

    def copy_field(self, dst, src):
        self.check(self.lib.mm_copy_field(self.h, dst, src))

    def field_sums(self, field, ncomp):
        out = np.zeros(max(ncomp, 9))
        self.check(self.lib.mm_field_sums(self.h, field, _ptr(out)))
        return out[:ncomp].copy()

    def synchronize(self):
        self.check(self.lib.mm_synchronize(self.h))

    def device_bytes(self):
        return int(self.lib.mm_device_bytes(self.h))

    # -- compute -----------------------------------------------------------
    def set_symbols(self, axis_tab, threshold):
        t = np.ascontiguousarray(axis_tab, dtype=np.float64)
        self.check(self.lib.mm_set_symbols(self.h, _ptr(t), float(threshold)))

    def local_sweeps(self, material, rho, tol, max_sweeps, phi_scale, want_points=False):
        st = LocalStatsC()
        self.check(self.lib.mm_local_sweeps(self.h, int(material), float(rho), float(tol),
                                            int(max_sweeps), float(phi_scale),
                                            1 if want_points else 0, ctypes.byref(st)))
        return st

    def download_points(self):
        res = np.empty(self.npts)
        nsw = np.empty(self.npts, dtype=np.int64)
        ok = np.empty(self.npts, dtype=np.uint8)
        self.check(self.lib.mm_download_points(self.h, _ptr(res), _ptr(nsw), _ptr(ok),
                                               self.npts))
        return res, nsw, ok.astype(bool)

    def set_lce(self, **kw):
        p = LCEParamsC(**kw)
        self.check(self.lib.mm_set_lce(self.h, ctypes.byref(p)))

    def prepare_frozen(self):
        self.check(self.lib.mm_prepare_frozen(self.h))

    def project(self, rho, u_mean):
        um = np.ascontiguousarray(u_mean, dtype=np.float64).reshape(-1)
        self.check(self.lib.mm_project(self.h, float(rho), _ptr(um)))

    def project_update(self, rho, u_mean):
        um = np.ascontiguousarray(u_mean, dtype=np.float64).reshape(-1)
        st = UpdateStatsC()
        self.check(self.lib.mm_project_update(self.h, float(rho), _ptr(um), ctypes.byref(st)))
        return st

    def stencil(self, op):
        self.check(self.lib.mm_stencil(self.h, int(op)))

    def profile_enable(self, on=True):
        self.check(self.lib.mm_profile_enable(self.h, 1 if on else 0))

    def profile_read(self, reset=False):
        p = ProfileC()
        self.check(self.lib.mm_profile_read(self.h, ctypes.byref(p), 1 if reset else 0))
        return ({s: p.ms[i] for i, s in enumerate(STAGES)},
                {s: int(p.launches[i]) for i, s in enumerate(STAGES)})

    def set_option(self, option, value):
        self.check(self.lib.mm_set_option(self.h, int(option), int(value)))

    def project_residuals(self, rho, u_mean):
        um = np.ascontiguousarray(u_mean, dtype=np.float64).reshape(-1)
        st = UpdateStatsC()
        self.check(self.lib.mm_project_residuals(self.h, float(rho), _ptr(um), ctypes.byref(st)))
        return st

    def residuals_and_step(self, prm):
        """mm_residuals_and_step: prm is a StepParamsC; returns (result, local stats)."""
        res = StepResultC()
        ls = LocalStatsC()
        self.check(self.lib.mm_residuals_and_step(self.h, ctypes.byref(prm), ctypes.byref(res),
                                                  ctypes.byref(ls)))
        return res, ls

    def solve_fused(self, prm, max_outer):
        """mm_solve_fused: returns (result, history (iterations, 4), status);
        a diverged run returns MM_ERR_DIVERGED with the result filled."""
        res = SolveResultC()
        hist = np.zeros((max(int(max_outer), 1), 4))
        rc = self.lib.mm_solve_fused(self.h, ctypes.byref(prm), ctypes.byref(res), _ptr(hist))
        if rc not in (MM_OK, MM_ERR_DIVERGED):
            self.check(rc)
        n = int(res.iterations) - (1 if res.diverged else 0)
        msg = self.lib.mm_last_error(self.h).decode() if rc else ""
        return res, hist[:n].copy(), rc, msg

    def update_multiplier(self):
        st = UpdateStatsC()
        self.check(self.lib.mm_update_multiplier(self.h, ctypes.byref(st)))
        return st

    def update_and_sweep(self, material, rho_next, tol, max_sweeps, phi_scale, want_points=False):
        ls = LocalStatsC()
        us = UpdateStatsC()
        self.check(self.lib.mm_update_and_sweep(self.h, int(material), float(rho_next), float(tol),
                                                int(max_sweeps), float(phi_scale),
                                                1 if want_points else 0, ctypes.byref(ls),
                                                ctypes.byref(us)))
        return ls, us

    # -- slab decomposition ------------------------------------------------------
    def slab_buffer(self, which):
        ptr = ctypes.c_void_p()
        nbytes = ctypes.c_int64()
        self.check(self.lib.mm_slab_buffer(self.h, int(which), ctypes.byref(ptr),
                                           ctypes.byref(nbytes)))
        return ptr.value, nbytes.value

    # -- Bloch stability -----------------------------------------------------------
    def bloch_setup(self, Minv, Lmat, shift, bsq, live, rho, target):
        Minv = np.ascontiguousarray(Minv, dtype=np.float64)
        Lmat = np.ascontiguousarray(Lmat, dtype=np.float64)
        shift = np.ascontiguousarray(shift, dtype=np.float64)
        bsq = np.ascontiguousarray(bsq, dtype=np.float64)
        live = np.ascontiguousarray(live, dtype=np.uint8)
        self.check(self.lib.mm_bloch_setup(self.h, _ptr(Minv), _ptr(Lmat), _ptr(shift),
                                           _ptr(bsq), _ptr(live), float(rho), float(target)))

    def bloch_start(self, p):
        p = np.ascontiguousarray(p, dtype=np.complex128)
        self.check(self.lib.mm_bloch_start(self.h, _ptr(p)))

    def bloch_iterate(self, max_iter, tol_beta, tol_primal, floor, mu_rep):
        out = np.zeros(5)
        self.check(self.lib.mm_bloch_iterate(self.h, int(max_iter), float(tol_beta),
                                             float(tol_primal), float(floor), float(mu_rep),
                                             _ptr(out)))
        return float(out[0]), float(out[1]), int(out[2]), bool(out[3]), bool(out[4])

    def bloch_mode(self, shape):
        out = np.empty(shape, dtype=np.complex128)
        self.check(self.lib.mm_bloch_mode(self.h, _ptr(out)))
        return out

    def slab_set_peers(self, which, ptrs):
        arr = (ctypes.c_void_p * len(ptrs))(*[int(p) for p in ptrs])
        self.check(self.lib.mm_slab_set_peers(self.h, int(which), arr, len(ptrs)))

    def slab_ipc_handle(self, which):
        buf = ctypes.create_string_buffer(64)
        self.check(self.lib.mm_slab_ipc_handle(self.h, int(which), buf))
        return buf.raw

    def slab_open_peers(self, which, handles):
        blob = b"".join(handles)
        buf = ctypes.create_string_buffer(blob, len(blob))
        self.check(self.lib.mm_slab_open_peers(self.h, int(which), buf, len(handles)))

    def slab_step(self, step, rho, u_mean=None):
        sums = np.zeros(11)
        um = None
        if u_mean is not None:
            um = np.zeros(9)
            u = np.asarray(u_mean, dtype=np.float64).reshape(-1)
            um[: u.size] = u
        self.check(self.lib.mm_slab_step(self.h, int(step), float(rho),
                                         _ptr(um) if um is not None else None, _ptr(sums)))
        return sums

    def slab_field(self, which):
        """(device pointer of plane 0, component stride, components, ghost planes)."""
        base = ctypes.c_void_p()
        cs = ctypes.c_int64()
        nc = ctypes.c_int()
        g = ctypes.c_int()
        self.check(self.lib.mm_slab_field(self.h, int(which), ctypes.byref(base), ctypes.byref(cs),
                                          ctypes.byref(nc), ctypes.byref(g)))
        return base.value, cs.value, nc.value, g.value

    def slab_stream(self):
        st = ctypes.c_void_p()
        self.check(self.lib.mm_slab_stream(self.h, ctypes.byref(st)))
        return st.value


class DeviceArray:
    """__cuda_array_interface__ view of a device buffer owned by a Context
    (lets torch / NCCL move it without copies)."""

    def __init__(self, ptr, shape, typestr="<f8", owner=None):
        self.__cuda_array_interface__ = {"shape": tuple(int(x) for x in shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3}
        self._owner = owner
