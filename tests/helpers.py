"""Shared helpers of the parity tests: identical mesh configs for the oracle
(oracle/pyoracle.py) and the product (paper_2605_16684_b200/capi.py), and the
error norms the tolerances are stated in."""
import numpy as np

from oracle import pyoracle as po
from paper_2605_16684_b200 import capi


def both_configs(kind, *args, **kw):
    """(oracle MeshConfig, product MeshConfig) of the same mesh."""
    if kind == "bubble":
        return po.bubble_mesh_config(*args, **kw), capi.bubble_mesh_config(*args, **kw)
    if kind == "unit":
        return po.unit_mesh_config(*args), capi.mesh_config((1, 1, 1), args[0])
    if kind == "raw":
        return po.mesh_config(*args), capi.mesh_config(*args)
    raise ValueError(kind)


def settings_pair(dissipation=True, mode=0, f0=0.0, beta=0.0, y0=0.0):
    return (po.make_settings(dissipation, mode, f0, beta, y0),
            capi.Settings(int(dissipation), mode, f0, beta, y0))


def gas_pair(gravity=9.81):
    return po.default_gas(gravity), capi.Gas(1.4, 287.0, 1e5, gravity)


def scaled_error(got, want, scale):
    """max_v max|got_v - want_v| / S_v with S_v the abs-sum flux scale of the
    oracle: the magnitude of the terms the RHS adds up, which
    stays meaningful when the tendency itself is a near-perfect cancellation
    (hydrostatic states). Variables whose scale is 0 must match exactly."""
    worst = 0.0
    for v in range(5):
        d = float(np.abs(got[:, v].astype(np.float64) - want[:, v].astype(np.float64)).max())
        if scale[v] == 0.0:
            assert d == 0.0, f"variable {v}: scale 0 but diff {d}"
            continue
        worst = max(worst, d / scale[v])
    return worst


def max_rel_diff(a, b):
    """ladder.hpp:14-22 of the reference: max|a-b| / max|a|."""
    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    s = float(np.abs(a64).max())
    d = float(np.abs(a64 - b64).max())
    return d / s if s > 0 else d


def state_error(got, want):
    """per-variable max|dq_v| / max|q_v| (trajectory tolerance)."""
    out = []
    for v in range(5):
        s = float(np.abs(want[:, v].astype(np.float64)).max())
        d = float(np.abs(got[:, v].astype(np.float64) - want[:, v].astype(np.float64)).max())
        out.append(d / s if s > 0 else d)
    return out


# ---- sampled comparison on meshes too large to assemble on one CPU core ----------

def sample_ranges(ne, epb, runs, rng):
    """Element ranges [b, e) to check: first and last CTA (the last one is
    partial when epb does not divide ne), both sides of every step_swap run
    boundary, and random places."""
    groups = (ne + epb - 1) // epb
    picks = [(0, 3), (ne - 3, ne), ((groups - 1) * epb - 2, min(ne, (groups - 1) * epb + 2))]
    for r in range(1, runs):
        g0 = groups * r // runs
        picks.append((g0 * epb - 2, g0 * epb + 2))
    for b in rng.integers(0, ne - 3, 40):
        picks.append((int(b), int(b) + 3))
    return [(max(0, b), min(ne, e)) for b, e in picks]


def face_table(omesh):
    """The oracle mesh's Face records (mesh.hpp:35-41) as a structured array."""
    import ctypes as C
    p = omesh.o.f("mesh_faces")(omesh.h)
    dt = np.dtype([("minus_elem", "<i4"), ("plus_elem", "<i4"), ("dir", "u1"), ("minus_side", "u1"),
                   ("reflecting", "u1"), ("pad", "u1")])
    buf = (C.c_char * (omesh.nfaces * dt.itemsize)).from_address(C.addressof(p.contents))
    return np.frombuffer(buf, dtype=dt)


def check_samples(o, face_of, faces, q, got, ranges, tol):
    """Oracle RHS of the element ranges (assemble_rhs_rank, the neighbours'
    traces extracted from the full state like a rank's ghost traces) against
    the same elements of the GPU result."""
    slot = np.full(o.mesh.nfaces, -1, np.int32)
    want = np.zeros(q.shape, q.dtype)          # lazily committed; only the samples are touched
    worst, n = 0.0, 0
    for b, e in ranges:
        traces, used = [], []
        for el in range(b, e):
            for lf in range(6):
                fid = int(face_of[el, lf])
                f = faces[fid]
                if f["reflecting"] or slot[fid] >= 0:
                    continue
                am_minus = int(f["minus_elem"]) == el and int(f["minus_side"]) == lf % 2
                other = int(f["plus_elem"]) if am_minus else int(f["minus_elem"])
                if b <= other < e:
                    continue
                oside = (1 - int(f["minus_side"])) if am_minus else int(f["minus_side"])
                slot[fid] = len(traces)
                used.append(fid)
                traces.append(o.extract_trace(q, other, int(f["dir"]), oside))
        gt = np.ascontiguousarray(np.stack(traces)) if traces else np.zeros((1, 5, o.nq * o.nq), q.dtype)
        o.assemble_rhs_rank(q, want, 0.0, 1.0, b, e, slot, gt)
        scale = o.flux_scale_rank(q, b, e, slot, gt)
        worst = max(worst, scaled_error(got[b:e], want[b:e], scale))
        n += e - b
        slot[used] = -1
    assert worst <= tol, f"{n} sampled elements: scaled error {worst:.3e}"
    return worst, n
