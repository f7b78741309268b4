"""Quick device-side timing of the individual kernels (development aid; the
graded numbers come from bench.py)."""
import argparse
import json
import sys
import time

sys.path.insert(0, ".")
from paper_2605_16684_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--order", type=int, default=4)
ap.add_argument("--base", type=int, nargs=3, default=[3, 3, 3])
ap.add_argument("--refinement", type=int, default=5)
ap.add_argument("--precision", default="f64")
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()

out = {}
for prec in (8, 4):
    out[f"fma_peak_tflops_f{prec * 8}"] = capi.measure_fma_peak(0, prec)
mesh = capi.Mesh(capi.bubble_mesh_config(args.refinement, False, tuple(args.base)))
t0 = time.time()
s = capi.GpuSolver(mesh, args.order, args.precision)
s.init_case(capi.CASE_BUBBLE_SHARP)
out["setup_s"] = time.time() - t0
ne, n3 = mesh.ne, s.n3
dof = ne * n3
out.update(elements=ne, dof=dof, order=args.order, precision=args.precision)
dt = 1e-3
for path, name in ((capi.PATH_SPLIT, "split"), (capi.PATH_FUSED, "fused"), (capi.PATH_STAGE, "stage")):
    s.set_path(path)
    s.step(dt)          # warm-up
    s.sync()
    s.enable_timing(True)
    s.timers(reset=True)
    t0 = time.time()
    for _ in range(args.reps):
        s.step(dt, check_state=False)
    s.sync()
    wall = time.time() - t0
    t = s.timers(reset=True)
    s.enable_timing(False)
    n_rhs = 5 * args.reps
    out[name] = dict(
        wall_ms_per_step=1e3 * wall / args.reps,
        dof_rhs_per_s=dof * n_rhs / wall,
        volume_ms=1e3 * t["volume"] / n_rhs, surface_ms=1e3 * t["surface"] / n_rhs,
        update_ms=1e3 * t["update"] / n_rhs,
        ns_per_element_rhs=1e9 * wall / n_rhs / ne)
print(json.dumps(out, indent=1))
