"""Order / precision sweep of the step throughput (BASELINE.json configs[1]):
~1e8 DOF per order, FP64 and FP32. Development aid; prints one JSON line per
point."""
import json
import sys
import time

sys.path.insert(0, ".")
from paper_2605_16684_b200 import capi  # noqa: E402

# (order, base, refinement): SURVEY.md 8(d) config 2
POINTS = [(4, (3, 3, 3), 5), (5, (5, 5, 5), 4), (6, (1, 1, 1), 6), (7, (15, 15, 15), 2),
          (3, (2, 2, 2), 6), (2, (5, 5, 5), 5)]
only = [int(a) for a in sys.argv[1:]] or None
for order, base, ref in POINTS:
    if only and order not in only:
        continue
    for prec in ("f64", "f32"):
        mesh = capi.Mesh(capi.bubble_mesh_config(ref, False, base))
        s = capi.GpuSolver(mesh, order, prec)
        s.init_case(capi.CASE_BUBBLE_SHARP)
        dof = mesh.ne * s.n3
        dt = 1e-3
        row = dict(order=order, precision=prec, elements=mesh.ne, dof=dof)
        for path, name in ((capi.PATH_SPLIT, "split"), (capi.PATH_STAGE, "stage")):
            s.set_path(path)
            s.step(dt)
            s.sync()
            s.enable_timing(True)
            s.timers(reset=True)
            reps = 3
            t0 = time.time()
            for _ in range(reps):
                s.step(dt, check_state=False)
            s.sync()
            wall = time.time() - t0
            t = s.timers(reset=True)
            s.enable_timing(False)
            n = 5 * reps
            row[name] = dict(ms_step=round(1e3 * wall / reps, 3), gdof_s=round(dof * n / wall / 1e9, 3),
                             vol_ms=round(1e3 * t["volume"] / n, 3), surf_ms=round(1e3 * t["surface"] / n, 3),
                             upd_ms=round(1e3 * t["update"] / n, 3))
        print(json.dumps(row), flush=True)
        del s, mesh
