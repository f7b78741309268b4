"""Prints the GPU-vs-oracle error levels the test tolerances are set from."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle import pyoracle as po
from paper_2605_16684_b200 import capi
from helpers import both_configs, gas_pair, max_rel_diff, scaled_error, settings_pair

port = po.Oracle("port")
print("selftest f64", capi.selftest(0, 8))
print("selftest f32", capi.selftest(0, 4))
cases = [("bubble", (3, False), po.CASE_BUBBLE_SHARP, 0), ("bubble", (2, False), po.CASE_BUBBLE_SMOOTH, 0),
         ("bubble", (1, True), po.CASE_ENTROPY_TEST, 20240501), ("bubble", (2, True), po.CASE_ENTROPY_TEST, 5)]
for prec in ("f64", "f32"):
    for kind, margs, case, seed in cases:
        for order in (1, 2, 3, 4, 5, 6, 7):
            if order > 4 and margs[0] >= 3:
                continue
            for diss in (True, False):
                oc, cc = both_configs(kind, *margs)
                so, sc = settings_pair(diss)
                o = port.mesh(oc).solver(order, prec, settings=so)
                g = capi.GpuSolver(capi.Mesh(cc), order, prec, settings=sc)
                q = o.init_case(case, seed).copy()
                scale = o.flux_scale(q)
                want = o.assemble_rhs(q)
                wv = o.volume_rhs(q)
                out = [f"{prec} {kind}{margs} case{case} N={order} diss={int(diss)}"]
                for path in (capi.PATH_SPLIT, capi.PATH_FUSED, capi.PATH_STAGE):
                    g.set_path(path)
                    got = g.assemble_rhs(q)
                    per = [float(np.abs(got[:, v].astype(np.float64) - want[:, v]).max() / scale[v]) if scale[v] > 0 else 0.0
                           for v in range(5)]
                    out.append("path%d scaled %.2e (var %d) relmax %.2e" % (path, max(per), int(np.argmax(per)),
                                                                          max_rel_diff(want, got)))
                gv = g.volume_rhs(q)
                out.append("vol relmax %.2e scaled %.2e" % (max_rel_diff(wv, gv), scaled_error(gv, wv, scale)))
                print(" | ".join(out), flush=True)
