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
