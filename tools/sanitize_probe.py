import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2605_16684_b200 import capi
mesh = capi.Mesh(capi.bubble_mesh_config(1, False))
for prec in ("f64", "f32"):
    for order in (2, 4, 5):
        s = capi.GpuSolver(mesh, order, prec, ranks=2)
        s.init_case(capi.CASE_BUBBLE_SMOOTH)
        for path in (capi.PATH_SPLIT, capi.PATH_FUSED, capi.PATH_STAGE):
            s.set_path(path)
            s.step(1e-3)
        print(prec, order, float(np.abs(s.get_state()).max()), s.compute_dt(0.5), s.total_entropy())
