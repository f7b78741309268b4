"""Total-entropy evolution of BASELINE.json configs[0] (sharp rising bubble,
N=4, 8^3 elements, dt = compute_dt(0.5)) on the GPU (stage path, device
reductions) next to the reference's CPU solver, step by step. Prints a table
and the largest deviations; profiles/r1_entropy_evolution.txt is its output."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle import pyoracle as po  # noqa: E402
from paper_2605_16684_b200 import capi  # noqa: E402
from helpers import both_configs, gas_pair, settings_pair  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
every = int(sys.argv[2]) if len(sys.argv) > 2 else 10
kind = "reference" if po.reference_available() else "port"
ora = po.Oracle(kind)
oc, cc = both_configs("bubble", 3, False)
so, sc = settings_pair(True)
go, gc = gas_pair(9.81)
o = ora.mesh(oc).solver(4, "f64", gas=go, settings=so)
g = capi.GpuSolver(capi.Mesh(cc), 4, "f64", gas=gc, settings=sc)
g.set_path(capi.PATH_STAGE)
q0 = o.init_case(po.CASE_BUBBLE_SHARP).copy()
g.set_state(q0)
dt = o.compute_dt(0.5)
assert g.compute_dt(0.5) == dt
print(f"oracle: {kind}; dt = {dt!r}; {steps} LSRK steps")
print(f"{'step':>5s} {'eta CPU':>24s} {'eta GPU - CPU':>14s} {'prod CPU':>15s} {'prod GPU':>15s} "
      f"{'mass drift GPU':>15s} {'energy drift GPU':>16s} {'max|dq|/max|q|':>15s}")
eta0 = o.total_entropy(o.state.copy())
m0, e0 = g.quadrature_total(0), g.quadrature_total(4)
worst = dict(eta=0.0, prod=0.0, state=0.0)
for n in range(steps + 1):
    if n % every == 0:
        qs = o.state.copy()
        gs = g.get_state()
        eta_c, eta_g = o.total_entropy(qs), g.total_entropy()
        p_c = o.entropy_production(qs, o.assemble_rhs(qs))
        g.rhs(0.0, 1.0)                      # k <- RHS(q): the pair entropy_production reads
        p_g = g.entropy_production()
        dm = (g.quadrature_total(0) - m0) / m0
        de = (g.quadrature_total(4) - e0) / e0
        dq = max(float(np.abs(gs[:, v] - qs[:, v]).max()) / float(np.abs(qs[:, v]).max() + 1e-300)
                 for v in (0, 4))
        worst["eta"] = max(worst["eta"], abs(eta_g - eta_c) / abs(eta_c))
        if abs(p_c) > 0:
            worst["prod"] = max(worst["prod"], abs(p_g - p_c) / abs(p_c))
        worst["state"] = max(worst["state"], dq)
        print(f"{n:5d} {eta_c:24.16e} {eta_g - eta_c:14.3e} {p_c:15.7e} {p_g:15.7e} {dm:15.3e} {de:16.3e} {dq:15.3e}")
    if n < steps:
        o.step(dt)
        g.step(dt)
print(f"eta(t_end) - eta(0) CPU: {o.total_entropy(o.state.copy()) - eta0:.6e}")
print(f"largest deviations: total entropy {worst['eta']:.2e} relative, entropy production "
      f"{worst['prod']:.2e} relative, state (rho, E) {worst['state']:.2e} of max|q|")
