"""Host-side logic of the product (mesh, operators, partition, exchange plan,
GPU halo lists) against the oracle, and the C-ABI surface: the library loads
without a GPU and exports every symbol include/esdg_b200.h declares. No
compute entry point is called here. CPU only."""
import os
import re

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2605_16684_b200 import capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MESHES = [
    (po.bubble_mesh_config(3), capi.bubble_mesh_config(3)),
    (po.bubble_mesh_config(1, True), capi.bubble_mesh_config(1, True)),
    (po.mesh_config((3, 1, 2), 1, (0., 0., 0.), (3., 1., 2.), (0, 1, 0)),
     capi.mesh_config((3, 1, 2), 1, (0., 0., 0.), (3., 1., 2.), (0, 1, 0))),
    (po.mesh_config((1, 1, 1), 0), capi.mesh_config((1, 1, 1), 0)),
    (po.mesh_config((5, 3, 2), 0, bc=(1, 1, 1)), capi.mesh_config((5, 3, 2), 0, bc=(1, 1, 1))),
    (po.mesh_config((12, 2, 1), 1, (0., 0., 0.), (4e7, 6e6, 3e4), (0, 1, 1)), capi.channel_mesh_config(1)),
]


def test_header_symbols_exported_and_bound():
    """Every function include/esdg_b200.h declares is exported by the shared
    library and has a ctypes signature (so the binding cannot drift)."""
    text = open(os.path.join(ROOT, "include", "esdg_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    declared = set(re.findall(r"\b(esdg_b200_[a-z0-9_]+)\s*\(", text))
    declared -= {"esdg_b200_exchange_fn"}
    assert len(declared) > 50
    lib = capi.lib()
    for name in sorted(declared):
        assert hasattr(lib, name), f"{name} not exported"
        assert name in capi.SIGNATURES, f"{name} has no ctypes signature"
    assert set(capi.SIGNATURES) <= declared
    assert lib.esdg_b200_abi_version() == 1


def test_no_silent_cpu_fallback():
    """Without a device every compute path must fail loudly."""
    if capi.lib().esdg_b200_device_count() > 0:
        pytest.skip("a GPU is present")
    mesh = capi.Mesh(capi.bubble_mesh_config(1))
    with pytest.raises(capi.EsdgError):
        capi.GpuSolver(mesh, 4, "f64")
    with pytest.raises(capi.EsdgError):
        capi.measure_fma_peak(0, 8)


def test_product_never_imports_oracle():
    """oracle/ is test infrastructure: nothing under the package references it."""
    pkg = os.path.join(ROOT, "paper_2605_16684_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".hpp", ".h")) or f == "Makefile":
                src = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "pyoracle" not in src and "liboracle" not in src and "esdg_oracle" not in src, f
                assert "libesdg_ref" not in src, f


def test_operators_and_lsrk(port):
    for order in range(1, 8):
        for a, b in zip(port.reference_element(order), capi.reference_element(order)):
            assert np.array_equal(a, b)
    for a, b in zip(port.lsrk(), capi.lsrk_coefficients()):
        assert np.array_equal(a, b)
    with pytest.raises(capi.EsdgError):
        capi.reference_element(0)


@pytest.mark.parametrize("idx", range(len(MESHES)))
def test_mesh_and_plan_match_oracle(port, idx):
    oc, cc = MESHES[idx]
    mo, mc = port.mesh(oc), capi.Mesh(cc)
    assert (mo.ne, mo.nfaces) == (mc.ne, mc.nfaces)
    assert np.array_equal(mo.lattice, mc.lattice)
    assert np.array_equal(mo.faces, mc.faces)
    assert np.array_equal(mo.face_of, mc.face_of)
    # neighbour table is consistent with the face list
    nbr, faces, face_of = mc.neighbors, mc.faces, mc.face_of
    for e in range(mc.ne):
        for lf in range(6):
            me, pe, d, ms, refl = faces[face_of[e, lf]]
            assert d == lf // 2
            if refl:
                assert nbr[e, lf] == -1
            else:
                assert nbr[e, lf] == (pe if (me == e and ms == lf % 2) else me)
    for ranks in (1, 2, 3, 4, 8):
        if ranks > mo.ne:
            with pytest.raises(capi.EsdgError):
                capi.partition(mo.ne, ranks)
            continue
        assert np.array_equal(port.partition(mo.ne, ranks), capi.partition(mo.ne, ranks))
        a, b = mo.exchange_plan(ranks), mc.exchange_plan(ranks)
        for k in a:
            assert np.array_equal(a[k], b[k]), (k, ranks)


def test_mesh_rejects_bad_config():
    for cfg in (capi.mesh_config((0, 1, 1)), capi.mesh_config(refinement=-1), capi.mesh_config(refinement=21),
                capi.mesh_config(lo=(0, 0, 0), hi=(1, 0, 1))):
        with pytest.raises(capi.EsdgError):
            capi.Mesh(cfg)


@pytest.mark.parametrize("idx", [0, 1, 2, 5])
@pytest.mark.parametrize("world", [2, 3, 4])
def test_rank_halo_consistency(port, idx, world):
    """The GPU halo lists: every ghost face of rank A toward B appears in B's
    block toward A at the same position, pointing at the opposite side of the
    same face; local codes address the right elements."""
    oc, cc = MESHES[idx]
    mo, mc = port.mesh(oc), capi.Mesh(cc)
    if world > mc.ne:
        pytest.skip("more ranks than elements")
    face_of, faces, nbr = mo.face_of, mo.faces, mc.neighbors
    halos = [capi.rank_halo(mc, world, r) for r in range(world)]
    plan = mo.exchange_plan(world)
    assert [len(h["send_elem"]) for h in halos] == list(plan["ghost_count"])
    for r, h in enumerate(halos):
        b, e = h["begin"], h["end"]
        codes = h["nbr_local"]
        seen = set()
        for el in range(e - b):
            for lf in range(6):
                n, code = nbr[b + el, lf], codes[el, lf]
                if n < 0:
                    assert code == -1
                elif b <= n < e:
                    assert code == n - b
                else:
                    v = -2 - code
                    slot, am_minus = v >> 1, v & 1
                    assert h["send_elem"][slot] == el and h["send_face"][slot] == lf
                    me, pe, d, ms, refl = faces[face_of[b + el, lf]]
                    assert am_minus == int(me == b + el and ms == lf % 2)
                    seen.add(slot)
        assert seen == set(range(len(h["send_elem"])))
        assert sum(c for _, _, c in h["peers"]) == len(h["send_elem"])
        for peer, off, cnt in h["peers"]:
            hp = halos[peer]
            poff = [o for (p, o, c) in hp["peers"] if p == r]
            assert len(poff) == 1 and [c for (p, o, c) in hp["peers"] if p == r] == [cnt]
            for i in range(cnt):
                mine = face_of[b + h["send_elem"][off + i], h["send_face"][off + i]]
                theirs = face_of[hp["begin"] + hp["send_elem"][poff[0] + i], hp["send_face"][poff[0] + i]]
                assert mine == theirs
                assert h["send_face"][off + i] == hp["send_face"][poff[0] + i] ^ 1


def _primitives(q, gas, z):
    rho = q[0]
    u = q[1:4] / rho
    p = (gas.gamma - 1.0) * (q[4] - 0.5 * rho * float(u @ u) - rho * gas.gravity * z)
    return rho, u, p


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_baroclinic_jet_is_balanced(mode):
    """CASE_BAROCLINIC_JET (ours; Ullrich et al. 2015 as PAPER.md:465-472 runs
    it) is a steady state of the equations the RHS integrates: with v = w = 0
    and no x dependence that is hydrostatic balance dp/dz = -rho g and
    geostrophic balance dp/dy = -rho f u with the solver's own Coriolis
    parameter f = f0 + beta (y - y0) (physics.hpp:276-306). Checked pointwise
    with centred differences of the generator's pressure (host only)."""
    cfg = capi.channel_mesh_config(3)
    gas = capi.Gas(1.4, 287.0, 1e5, 9.81)
    st = capi.Settings(1, mode, 1e-4, 1.6e-11, 3e6)
    nopert = [0.0, -1.0, 0.0, 0.0, 0.0]

    def prim(x, y, z):
        return _primitives(capi.case_point(capi.CASE_BAROCLINIC_JET, cfg, gas, st, x, y, z, dparam=nopert), gas, z)

    rng = np.random.default_rng(5)
    umax = 0.0
    for _ in range(200):
        x, y, z = rng.uniform(0, 4e7), rng.uniform(2e5, 5.8e6), rng.uniform(50.0, 2.9e4)
        rho, u, p = prim(x, y, z)
        assert rho > 0 and p > 0 and u[1] == 0 and u[2] == 0
        umax = max(umax, abs(u[0]))
        f = 0.0 if mode == 0 else (1e-4 if mode == 1 else 1e-4 + 1.6e-11 * (y - 3e6))
        hz, hy = 1.0, 2e3      # truncation h^2 p''' / 6 is 2e-9 resp. 1e-12 relative
        dpdz = (prim(x, y, z + hz)[2] - prim(x, y, z - hz)[2]) / (2 * hz)
        dpdy = (prim(x, y + hy, z)[2] - prim(x, y - hy, z)[2]) / (2 * hy)
        assert abs(dpdz + rho * gas.gravity) <= 1e-7 * rho * gas.gravity
        # 1e-6 of the largest geostrophic term in the channel (rho f u ~ 4e-3 Pa/m)
        assert abs(dpdy + rho * f * u[0]) <= 1e-6 * 1.2 * 1.3e-4 * 35.0 + 1e-9
    assert 25.0 < umax < 36.0
    # the walls carry no jet, the surface is the p0 surface
    assert abs(prim(1e6, 0.0, 1.5e4)[1][0]) < 1e-12 and abs(prim(1e6, 6e6, 1.5e4)[1][0]) < 1e-10
    assert abs(prim(1e6, 2e6, 0.0)[2] - gas.p0) <= 1e-9 * gas.p0
    # the perturbation: 1 m/s of zonal wind at (2000 km, 2500 km)
    q0 = capi.case_point(capi.CASE_BAROCLINIC_JET, cfg, gas, st, 2e6, 2.5e6, 1e4, dparam=nopert)
    q1 = capi.case_point(capi.CASE_BAROCLINIC_JET, cfg, gas, st, 2e6, 2.5e6, 1e4)
    assert abs((q1[1] - q0[1]) / q0[0] - 1.0) < 1e-12 and q1[0] == q0[0]


def test_library_is_a_product_build():
    """The tuning hooks are compile-time switches (make EXTRA=-DESDG_TUNE_...);
    the library the tests, smoke() and bench.py load must not carry any of
    them. (The ladder rungs are run-time selectable instances, not switches.)
    The Makefile records the flags of the last build and rebuilds everything
    when they change."""
    flags = open(os.path.join(capi.CSRC, "build", ".flags")).read()
    assert "ESDG_LADDER" not in flags and "ESDG_TUNE" not in flags, flags
    assert "arch=compute_100a,code=sm_100a" in flags and "-lineinfo" in flags


def test_lsrk_temporal_order():
    """acceptance.cpp:363-392 (criterion 10): lsrk_step with the exported
    Carpenter-Kennedy coefficients integrates q' = -q to t = 1 with observed
    order 4.0 +- 0.1 between dt = 0.1, 0.05, 0.025, 0.0125."""
    a, b, c = capi.lsrk_coefficients()
    assert a[0] == 0.0 and c[0] == 0.0

    def run(dt):
        q, k = 1.0, 0.0
        for _ in range(int(round(1.0 / dt))):
            for s in range(5):      # time_integration.hpp:43-49
                k = a[s] * k + dt * (-q)
                q += b[s] * k
        return abs(q - np.exp(-1.0))

    errs = [run(dt) for dt in (0.1, 0.05, 0.025, 0.0125)]
    orders = [np.log2(errs[i] / errs[i + 1]) for i in range(3)]
    assert min(orders) >= 3.9 and max(orders) <= 4.1, orders
