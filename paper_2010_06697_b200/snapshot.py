"""Solver-state snapshots (SPEC.md cli-io write_snapshot /
read_snapshot and admm-core "Field snapshot format").

A snapshot is two files written next to each other:

* ``<stem>.bin``  -- raw little-endian float64 arrays, concatenated in the
  order the sidecar lists them (fields in the reference's AoS layout,
  ``grid.shape + component shape``), then the residual history as an
  (n, 6) table;
* ``<stem>.meta`` -- a plain-text ``key = value`` sidecar: format version,
  grid dims, L, component order and transform convention, the scalar state
  (rho, counters, r_d_prev, u_mean, printed with 17 significant digits) and,
  per array, its name, shape and byte offset.

``read_snapshot(write_snapshot(s))`` reproduces every array and scalar bit
for bit.  Both files are written to temporaries and renamed, so an
interrupted write never leaves a partial snapshot.  A truncated or corrupt
``.bin`` raises SnapshotError with the byte offset at which reading failed;
a different format version is refused by name.

Device-resident states are read through their attributes (one D2H per
field); a loaded state is a host state that the next solve uploads.
"""

from __future__ import annotations

import os

import numpy as np

from .errors import SnapshotError
from .grid import Grid
from .solver import ADMMState, Residuals

__all__ = ["FORMAT_VERSION", "write_snapshot", "read_snapshot"]

FORMAT_VERSION = "mm-snapshot/1"
_FIELDS = ("F", "grad_u", "lam", "u_tilde", "prev_F")


def _fmt(x: float) -> str:
    return repr(float(x))  # shortest repr round-trips a double exactly


def _arrays(state: ADMMState):
    out = []
    for name in _FIELDS:
        v = getattr(state, name)
        if v is not None:
            out.append((name, np.asarray(v, dtype=float)))
    for group in ("internal", "prev_internal"):
        d = getattr(state, group)
        if d:
            for k in sorted(d):
                out.append((f"{group}.{k}", np.asarray(d[k], dtype=float)))
    hist = np.array([[float(r.outer_iter), r.r_p, r.r_d, r.r_l, r.rho, r.wall_ms]
                     for r in state.history], dtype=float).reshape(-1, 6)
    out.append(("history", hist))
    return out


def _atomic_write(path: str, data: bytes):
    tmp = path + ".tmp"
    with open(tmp, "wb") as f:
        f.write(data)
        f.flush()
        os.fsync(f.fileno())
    os.replace(tmp, path)


def write_snapshot(state: ADMMState, stem: str, grid: Grid | None = None) -> str:
    """Write ``<stem>.bin`` / ``<stem>.meta``; returns the stem."""
    stem = os.fspath(stem)
    arrays = _arrays(state)
    lines = [f"format = {FORMAT_VERSION}",
             "byte_order = little", "dtype = float64",
             "layout = grid axes row-major, components innermost (AoS)",
             "transform = unnormalised forward DFT, xi = pi m / L, m in [-n/2, n/2)"]
    if grid is not None:
        lines += [f"dim = {grid.dim}", f"n = {grid.n}", f"length = {_fmt(grid.length)}"]
    lines += [f"rho = {_fmt(state.rho)}", f"outer_iter = {int(state.outer_iter)}",
              f"total_sweeps = {int(state.total_sweeps)}", f"r_d_prev = {_fmt(state.r_d_prev)}",
              "u_mean = " + " ".join(_fmt(v) for v in np.asarray(state.u_mean).ravel()),
              f"u_mean_shape = {' '.join(str(s) for s in np.asarray(state.u_mean).shape)}"]
    blobs = []
    offset = 0
    for name, a in arrays:
        b = np.ascontiguousarray(a, dtype="<f8").tobytes()
        lines.append(f"array = {name} {offset} {len(b)} {' '.join(str(s) for s in a.shape)}")
        blobs.append(b)
        offset += len(b)
    lines.append(f"total_bytes = {offset}")
    _atomic_write(stem + ".bin", b"".join(blobs))
    _atomic_write(stem + ".meta", ("\n".join(lines) + "\n").encode())
    return stem


def _parse_meta(path: str) -> tuple[dict, list]:
    try:
        with open(path, encoding="utf-8") as f:
            text = f.read()
    except OSError as e:
        raise SnapshotError(f"cannot read snapshot metadata {path}: {e}") from e
    meta, arrays = {}, []
    for ln, line in enumerate(text.splitlines(), 1):
        if not line.strip():
            continue
        if " = " not in line:
            raise SnapshotError(f"{path}:{ln}: malformed line {line!r}")
        key, val = line.split(" = ", 1)
        if key == "array":
            parts = val.split()
            if len(parts) < 3:
                raise SnapshotError(f"{path}:{ln}: malformed array entry")
            arrays.append((parts[0], int(parts[1]), int(parts[2]),
                           tuple(int(s) for s in parts[3:])))
        else:
            meta[key] = val
    if meta.get("format") != FORMAT_VERSION:
        raise SnapshotError(f"unsupported snapshot version {meta.get('format')!r} "
                            f"(this build reads {FORMAT_VERSION!r})")
    return meta, arrays


def read_snapshot(stem: str) -> ADMMState:
    """Load a snapshot written by write_snapshot (bit-exact)."""
    stem = os.fspath(stem)
    meta, entries = _parse_meta(stem + ".meta")
    try:
        with open(stem + ".bin", "rb") as f:
            blob = f.read()
    except OSError as e:
        raise SnapshotError(f"cannot read snapshot data {stem}.bin: {e}", offset=0) from e
    total = int(meta.get("total_bytes", -1))
    if total != len(blob):
        raise SnapshotError(f"{stem}.bin holds {len(blob)} bytes, metadata says {total}",
                            offset=min(len(blob), max(total, 0)))
    fields, internal, prev_internal, hist = {}, {}, {}, None
    for name, off, nbytes, shape in entries:
        need = int(np.prod(shape)) * 8 if shape else 8
        if off + nbytes > len(blob) or nbytes != need:
            raise SnapshotError(f"array {name!r} at offset {off}: {nbytes} bytes do not fit "
                                f"shape {shape} / file of {len(blob)} bytes", offset=off)
        a = np.frombuffer(blob, dtype="<f8", count=nbytes // 8, offset=off).astype(float)
        a = a.reshape(shape)
        if name == "history":
            hist = a
        elif name.startswith("internal."):
            internal[name.split(".", 1)[1]] = a
        elif name.startswith("prev_internal."):
            prev_internal[name.split(".", 1)[1]] = a
        elif name in _FIELDS:
            fields[name] = a
        else:
            raise SnapshotError(f"unknown array {name!r}", offset=off)
    try:
        u_mean = np.array([float(v) for v in meta["u_mean"].split()])
        u_mean = u_mean.reshape(tuple(int(s) for s in meta["u_mean_shape"].split()))
        history = [Residuals(int(r[0]), float(r[1]), float(r[2]), float(r[3]), float(r[4]),
                             float(r[5])) for r in (hist if hist is not None else [])]
        st = ADMMState(u_mean=u_mean, u_tilde=fields.get("u_tilde"), grad_u=fields.get("grad_u"),
                       F=fields.get("F"), lam=fields.get("lam"), internal=internal,
                       rho=float(meta["rho"]), outer_iter=int(meta["outer_iter"]),
                       r_d_prev=float(meta["r_d_prev"]), total_sweeps=int(meta["total_sweeps"]),
                       history=history, prev_F=fields.get("prev_F"),
                       prev_internal=prev_internal or None)
    except (KeyError, ValueError) as e:
        raise SnapshotError(f"snapshot metadata incomplete: {e}") from e
    return st
