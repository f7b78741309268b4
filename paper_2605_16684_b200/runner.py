"""run_case on the GPU solver: the step loop and the output files of the
reference's runner (core/src/runner.cpp:135-269) driven through the C ABI.

    python -m paper_2605_16684_b200.runner --case bubble --order 4 \
        --refinement 3 --steps 100 --output-cadence 10 --out run_out

Writes, with the reference's file names and columns (runner.cpp:205-267):
  conservation.csv  step,time,mass,energy,mass_drift,energy_drift
  entropy.csv       step,time,total_entropy,entropy_production
  throughput.csv    elements,steps,wall_time_s,element_steps_per_s
  roofline.csv      kernel,ai,gflops,fraction_of_roof
  manifest.txt      the run's parameters and a "# ---- run summary ----" block

The samples use the device reductions (K6), so nothing but one double per
element leaves the GPU between steps. The mesh/case tables are this
repository's (bubble: tests/test_helpers.hpp:10-21 and cases.hpp:43-69;
channel: config.cpp:84-95 with the surrogate initial state of
csrc/host/cases.cpp -- the reference ships none), and theta_slice() writes
slices/theta_y0_<step>.csv like runner.cpp:78-123. The config-file parser is
not reproduced here: the reference's own runner.cpp + config.cpp compile
unmodified against GpuSolver (oracle/Makefile, tests/test_reference_swap.py)
and are the value-checked route for configuration files.
"""
from __future__ import annotations

import argparse
import os
import time

import numpy as np

from . import capi


def work_model(nq: int, bytes_per_real: int) -> dict:
    """PerfRecord flop/byte model (diagnostics.cpp:33-81) per element per RHS."""
    n2, n3, h = nq * nq, nq ** 3, nq // 2
    return {
        "volume": (n3 * (189 * h + 205), (11 * n3 + n2) * bytes_per_real),
        "surface": (843 * n2, 66 * n2 * bytes_per_real),
        "update": (10 * n3, 15 * n3 * bytes_per_real),
    }


def theta_slice(solver, mesh, gas, order):
    """write_theta_slice (runner.cpp:78-123): potential temperature on the node
    plane closest to y = 0 (or to the mid-plane when 0 lies outside the box),
    rows (x, z, theta) sorted by (z, x). Evaluated on the host in 64-bit from
    the downloaded state, like the reference."""
    cfg, nq = mesh.cfg, order + 1
    lo, hi = np.array(cfg.lo[:]), np.array(cfg.hi[:])
    cells = np.array(cfg.base[:], np.int64) << cfg.refinement
    delta = (hi - lo) / cells
    ycut = 0.0 if lo[1] <= 0.0 < hi[1] else 0.5 * (lo[1] + hi[1])
    lat = mesh.lattice
    y_lo = lo[1] + lat[:, 1] * delta[1]
    cut = np.nonzero((y_lo <= ycut) & (ycut < y_lo + delta[1]))[0]
    xi = capi.reference_element(order)[0]

    def coord(e, d, r):   # mesh.hpp:73-77
        return lo[d] + (lat[e, d][:, None] + 0.5 * (r[None, :] + 1.0)) * delta[d]

    yn = coord(cut, 1, xi)                                   # [cut, nq]
    b_best = np.abs(yn - ycut).argmin(axis=1)                # first minimum, like the reference
    q = solver.get_state().astype(np.float64)[cut].reshape(len(cut), 5, nq, nq, nq)   # [e, v, c, b, a]
    ph = solver.get_phi().astype(np.float64)[cut].reshape(len(cut), nq, nq, nq)
    idx = np.arange(len(cut))
    qs, phs = q[idx, :, :, b_best, :], ph[idx, :, b_best, :]  # [e, v, c, a], [e, c, a]
    rho = qs[:, 0]
    ke = 0.5 * (qs[:, 1] ** 2 + qs[:, 2] ** 2 + qs[:, 3] ** 2) / rho
    p = (gas.gamma - 1.0) * (qs[:, 4] - ke - rho * phs)
    temp = p / (rho * gas.R)
    cp = gas.gamma * gas.R / (gas.gamma - 1.0)
    theta = temp * (gas.p0 / p) ** (gas.R / cp)
    x = np.broadcast_to(coord(cut, 0, xi)[:, None, :], theta.shape)
    z = np.broadcast_to(coord(cut, 2, xi)[:, :, None], theta.shape)
    rows = np.stack([x.ravel(), z.ravel(), theta.ravel()], axis=1)
    return rows[np.lexsort((rows[:, 2], rows[:, 0], rows[:, 1]))]


def run_case(case="bubble", order=4, refinement=3, base=None, precision="f64", courant=0.5,
             steps=100, output_cadence=10, out_dir="run_out", path=capi.PATH_SPLIT,
             peak_gflops=None, peak_gbps=None, device=0, slices=True) -> dict:
    os.makedirs(out_dir, exist_ok=True)
    if slices:
        os.makedirs(os.path.join(out_dir, "slices"), exist_ok=True)
    if case == "bubble":
        cfg = capi.bubble_mesh_config(refinement, False, tuple(base or (1, 1, 1)))
        settings, case_id = capi.Settings(1, 0, 0.0, 0.0, 0.0), capi.CASE_BUBBLE_SHARP
    elif case == "baroclinic":
        cfg = capi.channel_mesh_config(refinement, tuple(base or (12, 2, 1)))
        settings, case_id = capi.Settings(1, 2, 1e-4, 1.6e-11, 3e6), capi.CASE_BAROCLINIC_JET
    else:
        raise ValueError(f"unknown case {case!r}")
    mesh = capi.Mesh(cfg)
    solver = capi.GpuSolver(mesh, order, precision, settings=settings, devices=[device])
    solver.set_path(path)
    solver.init_case(case_id)
    dt = solver.compute_dt(courant)
    digits = 17 if solver.prec == 8 else 9

    samples, entropy_rows = [], []

    def sample(step, t):
        mass, energy = solver.quadrature_total(0), solver.quadrature_total(4)
        eta = solver.total_entropy()
        solver.rhs(0.0, 1.0)            # k <- RHS(q): the pair entropy_production reads
        prod = solver.entropy_production()
        samples.append((step, t, mass, energy))
        entropy_rows.append((step, t, eta, prod))
        if slices:
            with open(os.path.join(out_dir, "slices", f"theta_y0_{step}.csv"), "w") as f:
                f.write("x,z,theta\n")
                for r in theta_slice(solver, mesh, solver.gas, order):
                    f.write(",".join(f"{v:.{digits}g}" for v in r) + "\n")

    status, t = "ok", 0.0
    secs = {"volume": 0.0, "surface": 0.0, "update": 0.0}
    solver.enable_timing(True)
    solver.timers(reset=True)
    wall, done = 0.0, 0
    try:
        sample(0, 0.0)
        solver.timers(reset=True)       # the samples' RHS calls are not the run's
        for step in range(1, steps + 1):
            t0 = time.perf_counter()
            solver.step(dt, check_state=True)
            solver.sync()
            wall += time.perf_counter() - t0
            done, t = step, step * dt
            if (output_cadence > 0 and step % output_cadence == 0) or step == steps:
                timers = solver.timers()
                sample(step, t)
                solver.timers(reset=True)
                for k in secs:
                    secs[k] += timers[k]
    except capi.NonPhysicalState as exc:
        status = f"nonphysical: {exc}"

    def fmt(x):
        return f"{x:.{digits}g}" if isinstance(x, float) else str(x)

    def write_csv(name, header, rows):
        with open(os.path.join(out_dir, name), "w") as f:
            f.write(header + "\n")
            for r in rows:
                f.write(",".join(fmt(v) for v in r) + "\n")

    m0, e0 = samples[0][2], samples[0][3]
    write_csv("conservation.csv", "step,time,mass,energy,mass_drift,energy_drift",
              [(s, tt, m, e, abs(m - m0) / abs(m0), abs(e - e0) / abs(e0)) for s, tt, m, e in samples])
    write_csv("entropy.csv", "step,time,total_entropy,entropy_production", entropy_rows)
    write_csv("throughput.csv", "elements,steps,wall_time_s,element_steps_per_s",
              [(mesh.ne, done, wall, mesh.ne * done / wall if wall > 0 else 0.0)])
    rb = solver.prec
    if peak_gflops is None:
        peak_gflops = 1e3 * capi.measure_fma_peak(device, rb)
    if peak_gbps is None:
        peak_gbps = 6456.5
    rows, model, n_rhs = [], work_model(order + 1, rb), 5 * done
    if path == capi.PATH_STAGE:
        # one kernel per stage: its time is booked under "volume"
        model = {"volume": tuple(sum(model[k][i] for k in model) for i in (0, 1))}
    elif path == capi.PATH_FUSED:
        model["volume"] = tuple(model["volume"][i] + model["surface"][i] for i in (0, 1))
    names = {capi.PATH_STAGE: {"volume": "stage (volume+surface+update)"},
             capi.PATH_FUSED: {"volume": "fused (volume+surface)"}}.get(path, {})
    for k in ("volume", "surface", "update"):
        s = secs.get(k, 0.0)
        if s <= 0.0 or k not in model:
            continue
        flops, nbytes = (v * mesh.ne * n_rhs for v in model[k])
        ai, gflops = flops / nbytes, flops / s / 1e9
        rows.append((names.get(k, k), ai, gflops, gflops / min(peak_gflops, ai * peak_gbps)))
    write_csv("roofline.csv", "kernel,ai,gflops,fraction_of_roof", rows)
    drift_m = max(abs(m - m0) / abs(m0) for _, _, m, _ in samples)
    drift_e = max(abs(e - e0) / abs(e0) for _, _, _, e in samples)
    with open(os.path.join(out_dir, "manifest.txt"), "w") as f:
        for k, v in (("case", case), ("order", order), ("refinement", refinement),
                     ("base", " ".join(map(str, cfg.base))), ("precision", precision),
                     ("courant", courant), ("steps", steps), ("output_cadence", output_cadence),
                     ("peak_gflops", peak_gflops), ("peak_gbps", peak_gbps)):
            f.write(f"{k} = {v}\n")
        f.write("# ---- run summary ----\n")
        for k, v in (("elements", mesh.ne), ("dof_per_var", mesh.ne * solver.n3), ("dt", dt),
                     ("steps_completed", done), ("wall_seconds", wall),
                     ("volume_seconds", secs.get("volume", 0.0)),
                     ("surface_seconds", secs.get("surface", 0.0)),
                     ("update_seconds", secs.get("update", 0.0)), ("rhs_calls", n_rhs),
                     ("mass_drift", drift_m), ("energy_drift", drift_e), ("status", status)):
            f.write(f"# {k} = {fmt(v)}\n")
    return dict(status=status, dt=dt, steps=done, wall_seconds=wall, mass_drift=drift_m,
                energy_drift=drift_e, entropy=entropy_rows, elements=mesh.ne)


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--case", default="bubble", choices=["bubble", "baroclinic"])
    ap.add_argument("--order", type=int, default=4)
    ap.add_argument("--refinement", type=int, default=3)
    ap.add_argument("--base", type=int, nargs=3, default=None)
    ap.add_argument("--precision", default="f64", choices=["f64", "f32"])
    ap.add_argument("--courant", type=float, default=0.5)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--output-cadence", type=int, default=10)
    ap.add_argument("--path", default="split", choices=["split", "fused", "stage"])
    ap.add_argument("--out", default="run_out")
    a = ap.parse_args()
    res = run_case(a.case, a.order, a.refinement, a.base, a.precision, a.courant, a.steps,
                   a.output_cadence, a.out,
                   {"split": capi.PATH_SPLIT, "fused": capi.PATH_FUSED, "stage": capi.PATH_STAGE}[a.path])
    print(f"{res['status']}: {res['steps']} steps of dt = {res['dt']:.6g} s on {res['elements']} elements in "
          f"{res['wall_seconds']:.3f} s; mass drift {res['mass_drift']:.2e}, energy drift "
          f"{res['energy_drift']:.2e}; eta {res['entropy'][0][2]:.16e} -> {res['entropy'][-1][2]:.16e}")


if __name__ == "__main__":
    main()
