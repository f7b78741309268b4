"""The reference's optimisation ladder (kernels.hpp:20-34, ladder.hpp:28-82) on the
GPU: device time of the volume kernel of every KernelVariant at BASELINE.json
configs[1] (N = 4, 884,736 elements, FP64), selected at run time with
esdg_b200_solver_set_variant. Development aid; prints one JSON line per rung."""
import json
import sys

sys.path.insert(0, ".")
from paper_2605_16684_b200 import capi  # noqa: E402

NAMES = ["baseline", "fused", "precompute", "logmean", "symmetric", "balanced"]
order = int(sys.argv[1]) if len(sys.argv) > 1 else 4
prec = sys.argv[2] if len(sys.argv) > 2 else "f64"
mesh = capi.Mesh(capi.bubble_mesh_config(5, False, (3, 3, 3)))
s = capi.GpuSolver(mesh, order, prec)
s.set_path(capi.PATH_SPLIT)
s.init_case(capi.CASE_BUBBLE_SHARP)
q0 = s.get_state()
base = None
for v in range(6):
    s.set_variant(v)
    s.set_state(q0)
    s.step(1e-3)
    s.sync()
    s.enable_timing(True)
    s.timers(reset=True)
    for _ in range(2):
        s.step(1e-3, check_state=False)
    s.sync()
    t = s.timers(reset=True)
    s.enable_timing(False)
    ms = 1e3 * t["volume"] / 10
    base = base or ms
    print(json.dumps(dict(variant=NAMES[v], order=order, precision=prec, volume_ms=round(ms, 3),
                          speedup_vs_baseline=round(base / ms, 2))), flush=True)
