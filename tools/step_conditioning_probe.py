"""Development aid: where does the FP32 k register of one LSRK step with matrix
dissipation differ from the oracle's? GPU FP32 and the FP32 oracle are both
compared with the FP64 oracle started from the same (FP32-representable) state."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle import pyoracle as po  # noqa: E402
from paper_2605_16684_b200 import capi  # noqa: E402
from helpers import both_configs, gas_pair, settings_pair  # noqa: E402

port = po.Oracle("port")
for order in (2, 4):
    for diss in (False, True):
        for path in (capi.PATH_SPLIT, capi.PATH_STAGE):
            oc, cc = both_configs("bubble", 1, True)
            so, sc = settings_pair(diss)
            go, gc = gas_pair(9.81)
            o32 = port.mesh(oc).solver(order, "f32", gas=go, settings=so)
            o64 = port.mesh(oc).solver(order, "f64", gas=go, settings=so)
            g = capi.GpuSolver(capi.Mesh(cc), order, "f32", gas=gc, settings=sc)
            g.set_path(path)
            q = o32.init_case(po.CASE_ENTROPY_TEST, 12345).copy()
            scale = o32.flux_scale(q)
            dt = float(np.float32(o32.compute_dt(0.4)))
            o32.state[:] = q
            o64.state[:] = q.astype(np.float64)
            g.set_state(q)
            o32.step(dt); o64.step(dt); g.step(dt)
            kg = g.get_state(capi.REG_K).astype(np.float64)
            k32 = np.asarray(o32.kreg, np.float64)
            k64 = np.asarray(o64.kreg, np.float64)
            def e(a, b):
                return max(float(np.abs(a[:, v] - b[:, v]).max()) / (dt * scale[v]) for v in range(5) if scale[v] > 0)
            # one RHS on identical input, for scale
            r32 = o32.assemble_rhs(q, np.zeros_like(q), 0.0, 1.0).astype(np.float64)
            r64 = o64.assemble_rhs(q.astype(np.float64), np.zeros(q.shape), 0.0, 1.0)
            rg = g.assemble_rhs(q, np.zeros_like(q), 0.0, 1.0).astype(np.float64)
            def er(a, b):
                return max(float(np.abs(a[:, v] - b[:, v]).max()) / scale[v] for v in range(5) if scale[v] > 0)
            print(f"N={order} diss={int(diss)} path={path}: k  gpu32-or32 {e(kg, k32):.2e}  gpu32-or64 {e(kg, k64):.2e}  or32-or64 {e(k32, k64):.2e}"
                  f" | rhs gpu32-or32 {er(rg, r32):.2e}  gpu32-or64 {er(rg, r64):.2e}  or32-or64 {er(r32, r64):.2e}")

# FP64: the same step from a state perturbed at the 1e-13 level (the size of the
# differences the first stage leaves between GPU and oracle): how much of it the
# k register of the whole step shows, with and without dissipation
rng = np.random.default_rng(7)
for order in (2, 4):
    for diss in (False, True):
        oc, cc = both_configs("bubble", 1, True)
        so, sc = settings_pair(diss)
        go, gc = gas_pair(9.81)
        oa = port.mesh(oc).solver(order, "f64", gas=go, settings=so)
        ob = port.mesh(oc).solver(order, "f64", gas=go, settings=so)
        g = capi.GpuSolver(capi.Mesh(cc), order, "f64", gas=gc, settings=sc)
        g.set_path(capi.PATH_STAGE)
        q = oa.init_case(po.CASE_ENTROPY_TEST, 12345).copy()
        scale = oa.flux_scale(q)
        dt = oa.compute_dt(0.4)
        oa.state[:] = q
        ob.state[:] = q * (1.0 + 1e-13 * rng.standard_normal(q.shape))
        g.set_state(q)
        oa.step(dt); ob.step(dt); g.step(dt)
        ka, kb = np.asarray(oa.kreg), np.asarray(ob.kreg)
        kg = g.get_state(capi.REG_K)
        e = lambda a, b: max(float(np.abs(a[:, v] - b[:, v]).max()) / (dt * scale[v]) for v in range(5) if scale[v] > 0)
        print(f"f64 N={order} diss={int(diss)}: k gpu-oracle {e(kg, ka):.2e} of dt*scale | oracle vs oracle from a 1e-13-perturbed state {e(kb, ka):.2e}")
