import sys, numpy as np
sys.path.insert(0, ".")
from paper_2605_16684_b200 import capi
st = capi.Settings(1, 2, 1e-4, 1.6e-11, 3e6)
for L in (1, 2, 3):
    mesh = capi.Mesh(capi.channel_mesh_config(L))
    g = capi.GpuSolver(mesh, 4, "f64", settings=st)
    g.set_path(capi.PATH_STAGE)
    g.init_case(capi.CASE_BAROCLINIC_JET, dparam=[0, -1, 0, 0, 0])
    q = g.get_state()
    rhs = g.assemble_rhs(q)
    print(L, mesh.ne, "max|rhs| per var", [float(np.abs(rhs[:, v]).max()) for v in range(5)],
          "max rho u", float(np.abs(q[:, 1]).max()), flush=True)
    if L == 2:
        dt = g.compute_dt(0.5)
        print("dt", dt)
        for i in range(200):
            g.step(dt)
        q2 = g.get_state()
        print("after 200 steps: max|v|", float(np.abs(q2[:, 2] / q2[:, 0]).max()), "max|w|",
              float(np.abs(q2[:, 3] / q2[:, 0]).max()), "max du", float(np.abs(q2[:, 1] / q2[:, 0] - q[:, 1] / q[:, 0]).max()))
