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
        print(prec, order, float(np.abs(s.get_state()).max()), s.compute_dt(0.5), s.total_entropy())
