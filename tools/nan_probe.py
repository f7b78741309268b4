import sys
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from oracle import pyoracle as po
from paper_2605_16684_b200 import capi
from helpers import both_configs, gas_pair, settings_pair
port = po.Oracle("port")
for order in (6, 7, 5):
    for ranks in (1, 2):
        for path in (capi.PATH_SPLIT, capi.PATH_FUSED):
            oc, cc = both_configs("bubble", 1, True)
            so, sc = settings_pair(True)
            go, gc = gas_pair(9.81)
            o = port.mesh(oc).solver(order, "f64", gas=go, settings=so)
            g = capi.GpuSolver(capi.Mesh(cc), order, "f64", gas=gc, settings=sc, ranks=ranks)
            g.set_path(path)
            q = o.init_case(po.CASE_ENTROPY_TEST, 1234).copy()
            scale = o.flux_scale(q)
            for a_old, a_new in ((0.0, 1.0), (0.0, 0.25), (0.7, 1.3)):
                out0 = (np.random.default_rng(1).standard_normal(q.shape) * scale[None, :, None]).astype(q.dtype)
                want = o.assemble_rhs(q, out0.copy(), a_old, a_new)
                got = g.assemble_rhs(q, out0.copy(), a_old, a_new)
                print(order, ranks, path, a_old, a_new, "nan in want", int(np.isnan(want).sum()), "nan in got", int(np.isnan(got).sum()),
                      "scale", scale, "maxdiff", float(np.nanmax(np.abs(got - want))), flush=True)
