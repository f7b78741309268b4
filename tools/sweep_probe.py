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


def work_model(nq, rb):
    """Algorithmic work per element per launch (the reference's PerfRecord
    model, core/src/diagnostics.cpp:33-81; the same closed forms as bench.py)."""
    n2, n3, h = nq * nq, nq ** 3, nq // 2
    return dict(volume_flops=n3 * (189 * h + 205), surface_flops=843 * n2,
                surface_bytes=66 * n2 * rb, update_bytes=15 * n3 * rb,
                stage_bytes=(6 + 5 + 5 + 5) * n3 * rb)  # q, phi, k in; k, q' out


try:
    with open("MEASURED_PEAKS.json") as f:
        HBM_GBS = float(json.load(f).get("hbm_gbs", 6650.0))
except OSError:
    HBM_GBS = 6650.0
FMA_PEAK = {p: capi.measure_fma_peak(0, p) for p in (8, 4)}  # TFLOP/s, measured in this run
# nominal: 148 SMs x 64 (128) lanes x 2 x 1.965 GHz
FMA_NOMINAL = {8: 148 * 64 * 2 * 1.965e9 / 1e12, 4: 148 * 128 * 2 * 1.965e9 / 1e12}
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
        # roofline fractions of this point: flux kernels against the CUDA-core
        # FMA peak (measured / nominal), surface and update against HBM
        rb = 8 if prec == "f64" else 4
        w = work_model(order + 1, rb)
        ne = mesh.ne
        st_tf = ne * (w["volume_flops"] + w["surface_flops"]) / (row["stage"]["vol_ms"] * 1e-3) / 1e12
        k1_tf = ne * w["volume_flops"] / (row["split"]["vol_ms"] * 1e-3) / 1e12
        row["roofline"] = dict(
            fma_peak_tflops=round(FMA_PEAK[rb], 2), fma_nominal_tflops=round(FMA_NOMINAL[rb], 2),
            hbm_peak_gbs=HBM_GBS,
            stage=dict(tflops=round(st_tf, 3), frac=round(st_tf / FMA_PEAK[rb], 4),
                       frac_nominal=round(st_tf / FMA_NOMINAL[rb], 4),
                       hbm_frac=round(ne * w["stage_bytes"] / (row["stage"]["vol_ms"] * 1e-3) / 1e9 / HBM_GBS, 4)),
            volume=dict(tflops=round(k1_tf, 3), frac=round(k1_tf / FMA_PEAK[rb], 4),
                        frac_nominal=round(k1_tf / FMA_NOMINAL[rb], 4)),
            surface_hbm_frac=round(ne * w["surface_bytes"] / (row["split"]["surf_ms"] * 1e-3) / 1e9 / HBM_GBS, 4),
            update_hbm_frac=round(ne * w["update_bytes"] / (row["split"]["upd_ms"] * 1e-3) / 1e9 / HBM_GBS, 4))
        print(json.dumps(row), flush=True)
        del s, mesh
