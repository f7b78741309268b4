"""Randomised parity sweep (development aid): orders 1..7, both precisions,
1..4 partitions, split, fused and stage paths, random (a_old, a_new), periodic
and walled meshes, against the CPU oracle with the tests' tolerances. On the
stage path (what bench.py times) a trial also takes one LSRK step through the
one-kernel-per-stage path and compares the k register and the state with the
oracle's Solver::step."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle import pyoracle as po  # noqa: E402
from paper_2605_16684_b200 import capi  # noqa: E402
from helpers import both_configs, gas_pair, settings_pair  # noqa: E402

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
port = po.Oracle("port")
worst = {"f64": 0.0, "f32": 0.0}
n = 0
for trial in range(int(sys.argv[2]) if len(sys.argv) > 2 else 60):
    order = int(rng.integers(1, 8))
    prec = "f64" if rng.random() < 0.6 else "f32"
    periodic = bool(rng.integers(0, 2))
    ranks = int(rng.integers(1, 5))
    diss = bool(rng.integers(0, 2))
    path = [capi.PATH_SPLIT, capi.PATH_FUSED, capi.PATH_STAGE][int(rng.integers(0, 3))]
    oc, cc = both_configs("bubble", 1 if order > 4 else int(rng.integers(1, 3)), periodic)
    so, sc = settings_pair(diss)
    go, gc = gas_pair(9.81)
    o = port.mesh(oc).solver(order, prec, gas=go, settings=so)
    g = capi.GpuSolver(capi.Mesh(cc), order, prec, gas=gc, settings=sc, ranks=ranks)
    g.set_path(path)
    q = o.init_case(po.CASE_ENTROPY_TEST, int(rng.integers(1, 1 << 30))).copy()
    scale = o.flux_scale(q)
    a_old = 0.0 if rng.random() < 0.3 else float(rng.uniform(-1.5, 1.5))
    a_new = float(rng.uniform(0.01, 2.0))
    out0 = (rng.standard_normal(q.shape) * scale[None, :, None]).astype(q.dtype)
    want = o.assemble_rhs(q, out0.copy(), a_old, a_new)
    got = g.assemble_rhs(q, out0.copy(), a_old, a_new)
    err = max(float(np.abs(got[:, v].astype(np.float64) - want[:, v]).max()) / (abs(a_new) * scale[v] + abs(a_old) * scale[v])
              for v in range(5) if scale[v] > 0)
    worst[prec] = max(worst[prec], err)
    tol = 2e-12 if prec == "f64" else 3e-5
    extra = ""
    if path == capi.PATH_STAGE:
        dt = o.compute_dt(0.4)
        dt = float(np.float32(dt)) if prec == "f32" else dt
        o.state[:] = q
        g.set_state(q)
        o.step(dt)
        g.step(dt)
        ek = max(float(np.abs(g.get_state(capi.REG_K)[:, v].astype(np.float64) - o.kreg[:, v]).max()) / (dt * scale[v])
                 for v in range(5) if scale[v] > 0)
        eq = max(float(np.abs(g.get_state()[:, v].astype(np.float64) - o.state[:, v]).max()) /
                 float(np.abs(o.state[:, v]).max()) for v in (0, 4))
        extra = f" | step: k {ek:.2e} of dt*scale, rho/E {eq:.2e} of max|q|"
        # The k register of a whole step is listed, not judged: with the matrix
        # dissipation a state difference of the size one stage leaves (1e-13 in
        # FP64, 1e-7 in FP32) comes back ~100 times larger in k -- the oracle
        # started from a state perturbed at that level moves as far, and the
        # reference's own FP32 build is 6e-4 ... 1.2e-3 of dt*scale from its
        # FP64 build (tools/step_conditioning_probe.py,
        # profiles/r2_step_conditioning.txt). Judged: the state after the step.
        err = max(err, eq)
    flag = "" if err <= tol else "   <-- above tolerance"
    print(f"N={order} {prec} periodic={int(periodic)} ranks={ranks} diss={int(diss)} path={path} "
          f"a_old={a_old:+.3f} a_new={a_new:.3f}: scaled error {err:.2e}{extra}{flag}")
    n += 1
print(f"{n} trials; worst scaled error f64 {worst['f64']:.2e}, f32 {worst['f32']:.2e}")
