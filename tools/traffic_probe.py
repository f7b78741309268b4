"""One LSRK step of one sweep point, for ncu: tools/collect_traffic.py wraps
this in `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum`.
usage: traffic_probe.py <order> <f64|f32> <bubble|baroclinic> <stage|fused|split>"""
import sys

sys.path.insert(0, ".")
from paper_2605_16684_b200 import capi  # noqa: E402

# (base, refinement) per order: SURVEY.md 8(d) config 2, ~1e8 DOF
POINTS = {2: ((5, 5, 5), 5), 3: ((2, 2, 2), 6), 4: ((3, 3, 3), 5), 5: ((5, 5, 5), 4), 6: ((1, 1, 1), 6),
          7: ((15, 15, 15), 2)}
order, prec, case, path = int(sys.argv[1]), sys.argv[2], sys.argv[3], sys.argv[4]
if case == "bubble":
    base, ref = POINTS[order]
    mesh = capi.Mesh(capi.bubble_mesh_config(ref, False, base))
    s = capi.GpuSolver(mesh, order, prec)
    s.init_case(capi.CASE_BUBBLE_SHARP)
else:
    mesh = capi.Mesh(capi.channel_mesh_config(5, (12, 2, 1)))
    s = capi.GpuSolver(mesh, order, prec, settings=capi.Settings(1, 2, 1e-4, 1.6e-11, 3e6))
    s.init_case(capi.CASE_BAROCLINIC_JET)
s.set_path({"stage": capi.PATH_STAGE, "fused": capi.PATH_FUSED, "split": capi.PATH_SPLIT}[path])
s.step(1e-3)
s.sync()
print("elements", mesh.ne)
