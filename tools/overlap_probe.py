"""Cost of splitting the one-pass stage kernel into interior and boundary
element groups (development aid): several partitions on ONE device, so the
halo path runs complete but nothing is gained from the overlap; what is
measured is the price of the second launch and of the scattered groups."""
import json
import sys
import time

sys.path.insert(0, ".")
from paper_2605_16684_b200 import capi  # noqa: E402

order = int(sys.argv[1]) if len(sys.argv) > 1 else 4
for ranks in (1, 2, 8):
    for overlap in (True, False):
        if ranks == 1 and not overlap:
            continue
        mesh = capi.Mesh(capi.bubble_mesh_config(5, False, (3, 3, 3)))
        s = capi.GpuSolver(mesh, order, "f64", ranks=ranks)
        s.set_path(capi.PATH_STAGE)
        s.set_overlap(overlap)
        s.init_case(capi.CASE_BUBBLE_SHARP)
        interior, total = s.overlap_elements()
        for _ in range(2):
            s.step(1e-3, check_state=False)
        s.sync()
        reps = 5
        t0 = time.time()
        for _ in range(reps):
            s.step(1e-3, check_state=False)
        s.sync()
        wall = (time.time() - t0) / reps
        print(json.dumps(dict(order=order, partitions=ranks, overlap=overlap, interior=interior,
                              elements=total, ms_step=round(1e3 * wall, 3),
                              gdof_s=round(total * s.n3 * 5 / wall / 1e9, 3))), flush=True)
        del s, mesh
