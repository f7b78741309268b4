import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2605_16684_b200 import capi
# 64 elements in 3 partitions: interior and boundary element groups both exist
# usage: sanitize_probe.py [orders, e.g. 2,4]
ORDERS = tuple(int(x) for x in sys.argv[1].split(",")) if len(sys.argv) > 1 else (2, 4, 5, 7)
mesh = capi.Mesh(capi.bubble_mesh_config(2, False))
for prec in ("f64", "f32"):
    for order in ORDERS:
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
        # independent states streamed through one solver (step_stream): three members
        # round-robin, upload of the next and download of the previous beside the step;
        # one partition (stage path) and three partitions (split path)
        for sp, path in ((s1, capi.PATH_STAGE), (s, capi.PATH_SPLIT)):
            sp.set_path(path)
            sp.init_case(capi.CASE_BUBBLE_SMOOTH)
            members = [sp.get_state() * (1.0 + 0.0) for _ in range(3)]
            outs = [np.empty_like(m) for m in members]
            sp.set_state(members[0])
            for call in range(6):
                nxt = members[(call + 1) % 3]
                prev = outs[(call - 1) % 3] if call > 0 else None
                sp.step_stream(1e-3, nxt, prev)
            sp.stream_collect(outs[5 % 3])
            print(prec, order, "stream", float(np.abs(outs[0]).max()), float(np.abs(outs[2]).max()))
