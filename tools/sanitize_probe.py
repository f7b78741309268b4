import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2605_16684_b200 import capi
# 64 elements in 3 partitions: interior and boundary element groups both exist
mesh = capi.Mesh(capi.bubble_mesh_config(2, False))
for prec in ("f64", "f32"):
    for order in (2, 4, 5, 7):
        s = capi.GpuSolver(mesh, order, prec, ranks=3)
        s.init_case(capi.CASE_BUBBLE_SMOOTH)
        for path in (capi.PATH_SPLIT, capi.PATH_FUSED, capi.PATH_STAGE):
            s.set_path(path)
            s.step(1e-3)
        q_host = s.get_state()
        s.step_swap(1e-3, q_host, q_host)          # one partition only: falls back here (3 partitions)
        s1 = capi.GpuSolver(mesh, order, prec)
        s1.set_path(capi.PATH_STAGE)
        s1.init_case(capi.CASE_BUBBLE_SMOOTH)
        s1.step_swap(1e-3, s1.get_state())         # last stage in runs of element groups
        print(prec, order, float(np.abs(s.get_state()).max()), s.compute_dt(0.5), s.total_entropy())
