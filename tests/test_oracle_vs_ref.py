"""The oracle restatement against the UNMODIFIED reference compiled from
/root/reference (oracle/_ref/libesdg_ref.so): bitwise, both precisions.
Skipped where the prebuilt reference library is absent. CPU only."""
import numpy as np
import pytest

from oracle import pyoracle as po


def test_mesh_plan_operators_bitwise(port, ref):
    for order in range(1, 9):
        for a, b in zip(port.reference_element(order), ref.reference_element(order)):
            assert np.array_equal(a, b)
    for nq in range(2, 10):
        for var in (0, 1):
            for a, b in zip(port.schedule(nq, var), ref.schedule(nq, var)):
                assert np.array_equal(a, b)
    for cfg in (po.bubble_mesh_config(2), po.bubble_mesh_config(1, True),
                po.mesh_config((3, 1, 2), 1, (0., 0., 0.), (3., 1., 2.), (0, 1, 0)),
                po.mesh_config((1, 1, 1), 0), po.mesh_config((5, 3, 2), 0, bc=(1, 1, 1))):
        mp, mr = port.mesh(cfg), ref.mesh(cfg)
        assert np.array_equal(mp.lattice, mr.lattice)
        assert np.array_equal(mp.faces, mr.faces)
        assert np.array_equal(mp.face_of, mr.face_of)
        assert mp.jacobian == mr.jacobian
        for ranks in (1, 2, 3, 4, 8):
            if ranks > mp.ne:
                continue
            a, b = mp.exchange_plan(ranks), mr.exchange_plan(ranks)
            for k in a:
                assert np.array_equal(a[k], b[k]), (k, ranks)


CASES = [(po.bubble_mesh_config(1, True), po.CASE_ENTROPY_TEST, 20240501),
         (po.bubble_mesh_config(1, False), po.CASE_BUBBLE_SMOOTH, 0),
         (po.mesh_config((2, 1, 3), 1, (0., 0., 0.), (4e3, 6e3, 3e3), (0, 1, 1)), po.CASE_ENTROPY_TEST, 7)]


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("order", [1, 2, 3, 4, 5, 7])
def test_solver_bitwise(port, ref, prec, order):
    for cfg, case, seed in CASES:
        for diss in (True, False):
            st = po.make_settings(diss, 2, 1e-4, 1.6e-11, 3e3)
            sp = port.mesh(cfg).solver(order, prec, settings=st)
            sr = ref.mesh(cfg).solver(order, prec, settings=st, ranks=2)
            qp, qr = sp.init_case(case, seed), sr.init_case(case, seed)
            assert np.array_equal(qp, qr) and np.array_equal(sp.phi, sr.phi)
            for k, v in sp.ops().items():
                assert np.array_equal(v, sr.ops()[k])
            assert np.array_equal(sp.assemble_rhs(qp.copy()), sr.assemble_rhs(qr.copy()))
            assert np.array_equal(sp.volume_rhs(qp.copy()), sr.volume_rhs(qr.copy()))
            o1 = sp.assemble_rhs(qp.copy())
            o2 = o1.copy()
            sp.assemble_rhs(qp.copy(), o1, -0.4, 0.3)
            sr.assemble_rhs(qr.copy(), o2, -0.4, 0.3)
            assert np.array_equal(o1, o2)
            dt = sp.compute_dt(0.5)
            assert dt == sr.compute_dt(0.5)
            for _ in range(2):
                sp.step(dt)
                sr.step(dt)
            assert np.array_equal(sp.state, sr.state)
            q = sp.state.copy()
            assert sp.total_entropy(q) == sr.total_entropy(q)
            assert sp.quadrature_total(q, 4) == sr.quadrature_total(q, 4)
            r = sp.assemble_rhs(q)
            assert sp.entropy_production(q, r) == sr.entropy_production(q, r)


def test_counter_closed_forms(ref):
    """test_kernels.cpp:95-162: the flop model's counters (BASELINE.md
    section 3) are what the reference actually counts."""
    mesh = ref.mesh(po.bubble_mesh_config(1, True))
    for order in (3, 4, 5):
        nq = order + 1
        n3, h = nq ** 3, nq // 2
        s = mesh.solver(order, "f64", settings=po.make_settings(False))
        q = s.init_case(po.CASE_ENTROPY_TEST, 5).copy()
        s.perf(reset=True)
        s.volume_rhs(q)
        p = s.perf()
        assert p["vol_flux"] == 3 * mesh.ne * n3 * h
        assert p["vol_log"] == 2 * mesh.ne * n3
        assert p["vol_div"] == mesh.ne * n3 * (23 + 24 * h)


def test_pointwise_bitwise(port, ref):
    sp = port.mesh(po.unit_mesh_config(0)).solver(1, "f64")
    sr = ref.mesh(po.unit_mesh_config(0)).solver(1, "f64")
    rng = np.random.default_rng(1)
    for _ in range(300):
        def draw():
            rho, u, p, phi = rng.uniform(0.5, 2), rng.uniform(-50, 50, 3), rng.uniform(5e4, 2e5), rng.uniform(0, 2e4)
            return np.array([rho, *(rho * u), p / 0.4 + 0.5 * rho * (u @ u) + rho * phi]), phi
        (qa, pa), (qb, pb) = draw(), draw()
        a8, b8 = sp.node_vals(qa, pa)[1], sp.node_vals(qb, pb)[1]
        assert np.array_equal(a8, sr.node_vals(qa, pa)[1])
        d = int(rng.integers(0, 3))
        assert np.array_equal(sp.ec_flux(a8, b8, d), sr.ec_flux(a8, b8, d))
        assert np.array_equal(sp.matrix_dissipation(a8, b8, d), sr.matrix_dissipation(a8, b8, d))
        x, y = rng.uniform(0.1, 3), rng.uniform(0.1, 3)
        y = x * (1 + rng.uniform(-1, 1) * 10.0 ** rng.integers(-9, 0))
        assert sp.log_mean(x, y, np.log(x), np.log(y)) == sr.log_mean(x, y, np.log(x), np.log(y))
