"""Replays one trial of tools/fuzz_parity.py (same seed, same draw sequence)
and repeats it with other values of a_new -- is an outlier driven by the state
or by the scaling? usage: fuzz_replay.py <seed> <trial index, 0-based>"""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle import pyoracle as po  # noqa: E402
from paper_2605_16684_b200 import capi  # noqa: E402
from helpers import both_configs, gas_pair, settings_pair  # noqa: E402

seed, target = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(seed)
port = po.Oracle("port")
for trial in range(target + 1):
    order = int(rng.integers(1, 8))
    prec = "f64" if rng.random() < 0.6 else "f32"
    periodic = bool(rng.integers(0, 2))
    ranks = int(rng.integers(1, 5))
    diss = bool(rng.integers(0, 2))
    path = [capi.PATH_SPLIT, capi.PATH_FUSED, capi.PATH_STAGE][int(rng.integers(0, 3))]
    level = 1 if order > 4 else int(rng.integers(1, 3))
    case_seed = int(rng.integers(1, 1 << 30))
    a_old = 0.0 if rng.random() < 0.3 else float(rng.uniform(-1.5, 1.5))
    a_new = float(rng.uniform(0.01, 2.0))
    ne = 8 ** level
    noise = rng.standard_normal((ne, 5, (order + 1) ** 3))
    if trial < target:
        continue
    oc, cc = both_configs("bubble", level, periodic)
    so, sc = settings_pair(diss)
    go, gc = gas_pair(9.81)
    o = port.mesh(oc).solver(order, prec, gas=go, settings=so)
    q = o.init_case(po.CASE_ENTROPY_TEST, case_seed).copy()
    scale = o.flux_scale(q)
    print(f"trial {trial}: N={order} {prec} periodic={int(periodic)} ranks={ranks} diss={int(diss)} path={path} "
          f"a_old={a_old:+.3f} a_new={a_new:.3f}")
    for r in (ranks, 1):
        for p in (path, capi.PATH_SPLIT):
            g = capi.GpuSolver(capi.Mesh(cc), order, prec, gas=gc, settings=sc, ranks=r)
            g.set_path(p)
            for an in (a_new, 1.0, 0.5, 0.0401, 1.7):
                out0 = (noise * scale[None, :, None]).astype(q.dtype)
                want = o.assemble_rhs(q, out0.copy(), a_old, an)
                got = g.assemble_rhs(q, out0.copy(), a_old, an)
                errs = [float(np.abs(got[:, v].astype(np.float64) - want[:, v]).max()) / ((abs(an) + abs(a_old)) * scale[v])
                        for v in range(5)]
                v = int(np.argmax(errs))
                e_at, n_at = np.unravel_index(int(np.abs(got[:, v].astype(np.float64) - want[:, v]).argmax()), got[:, v].shape)
                print(f"  ranks={r} path={p} a_new={an:.4f}: scaled error per variable " + " ".join(f"{e:.2e}" for e in errs)
                      + f" | worst at element {e_at}, node {n_at}, variable {v}")
