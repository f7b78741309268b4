"""Pins the oracle (the C restatement under oracle/) before it is trusted:
against the golden vectors generated from the reference itself
(tests/golden/make_golden.py), against the known-answer values of
BASELINE.md section 4 and against the reference's own physics KATs
(tests/test_physics.cpp). CPU only."""
import json
import math
import os

import numpy as np
import pytest

from oracle import pyoracle as po

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "golden.npz"))
with open(os.path.join(HERE, "golden", "kats.json")) as f:
    K = json.load(f)


def test_operators_match_reference_bitwise(port):
    for order in range(1, 8):
        x, w, d = port.reference_element(order)
        assert np.array_equal(x, G[f"lgl_nodes_{order}"])
        assert np.array_equal(w, G[f"lgl_weights_{order}"])
        assert np.array_equal(d, G[f"lgl_diff_{order}"])
    a, b, c = port.lsrk()
    assert np.array_equal(a, G["lsrk_a"]) and np.array_equal(b, G["lsrk_b"]) and np.array_equal(c, G["lsrk_c"])


def test_lgl_invariants(port):
    """reference_element.hpp:14-19: symmetric nodes, weights sum to 2, rows of
    D sum to 0, SBP property."""
    for order in range(1, 8):
        x, w, d = port.reference_element(order)
        assert x[0] == -1.0 and x[-1] == 1.0 and np.all(np.diff(x) > 0)
        assert np.array_equal(x, -x[::-1])
        assert abs(w.sum() - 2.0) < 1e-14
        assert np.abs(d.sum(axis=1)).max() < 1e-13
        q = np.diag(w) @ d
        b = np.zeros_like(q)
        b[0, 0], b[-1, -1] = -1.0, 1.0
        assert np.abs(q + q.T - b).max() < 1e-13


def test_rejects_bad_arguments(port):
    with pytest.raises(ValueError):
        port.reference_element(0)
    with pytest.raises(ValueError):
        port.reference_element(33)
    with pytest.raises(ValueError):
        port.schedule(1)
    with pytest.raises(ValueError):
        port.partition(4, 5)
    with pytest.raises(ValueError):
        port.partition(4, 0)
    with pytest.raises(ValueError):
        port.mesh(po.mesh_config((0, 1, 1)))


def test_schedule_pair_coverage(port):
    """test_schedule.cpp:27-101: every unordered pair has total weight 1."""
    for nq in range(2, 9):
        for variant in (0, 1):
            idx, hw, off = port.schedule(nq, variant)
            cover = np.zeros((nq, nq))
            for i in range(nq):
                part = idx[off[i]:off[i + 1]]
                assert list(part) == sorted(part)
                for j, h in zip(part, hw[off[i]:off[i + 1]]):
                    cover[min(i, j), max(i, j)] += 0.5 * h
            iu = np.triu_indices(nq, 1)
            assert np.all(cover[iu] == 1.0)
    idx, hw, off = port.schedule(5, 1)
    assert len(idx) == 10 and np.all(hw == 2)
    assert np.all(np.diff(off) == 2)


def test_partition_arithmetic(port):
    """test_partition.cpp:14-42."""
    assert list(port.partition(8, 2)) == [0, 4, 8]
    assert list(np.diff(port.partition(10, 4))) == [3, 3, 2, 2]


def test_exchange_plan_symmetry(port):
    """test_partition.cpp:44-73."""
    mesh = port.mesh(po.bubble_mesh_config(1, True))
    for ranks in (2, 3, 4, 8):
        plan = mesh.exchange_plan(ranks)
        gc = plan["ghost_count"]
        start = np.concatenate([[0], np.cumsum(gc)])
        by_rank = [plan["ghosts"][start[r]:start[r + 1]] for r in range(ranks)]
        for r in range(ranks):
            for face, peer, side, slot, inbox, outbox in by_rank[r]:
                match = [g for g in by_rank[peer] if g[0] == face]
                assert len(match) == 1
                g = match[0]
                assert g[1] == r and g[2] == 1 - side and g[4] == outbox and g[5] == inbox
        assert plan["interior_count"].sum() + gc.sum() // 2 == mesh.nfaces


def test_config1_known_answers(port):
    """BASELINE.md section 4 / kats.json: dt, RHS norms, conserved integrals,
    entropy and entropy production over 10 steps; bitwise state fingerprints."""
    c = K["config1_bubble_sharp_L3_N4_f64"]
    s = port.mesh(po.bubble_mesh_config(3)).solver(4, "f64")
    q = s.init_case(po.CASE_BUBBLE_SHARP)
    dt = s.compute_dt(0.5)
    assert dt == c["dt"] == 0.062160288912929212
    rhs0 = s.assemble_rhs(q.copy())
    assert [float(np.abs(rhs0[:, v]).max()) for v in range(5)] == c["rhs0_max_abs"]
    assert c["rhs0_max_abs"][3] == 0.030959300527197087
    assert "%016x" % po.fnv1a64(rhs0) == c["rhs0_fnv"]
    for row in c["steps"]:
        st = s.state.copy()
        rhs = s.assemble_rhs(st)
        assert s.quadrature_total(st, 0) == row["mass"] == 8559631581.0898724
        assert s.quadrature_total(st, 4) == row["energy"] == 1865806816191264.0
        assert s.total_entropy(st) == row["entropy"]
        assert s.entropy_production(st, rhs) == row["production"]
        assert "%016x" % po.fnv1a64(st) == row["q_fnv"]
        if row["step"] < 10:
            s.step(dt)
    assert np.array_equal(s.state[:16], G["config1_state10_elems0_16"])
    assert c["steps"][3]["production"] == -0.0008494687027185559
    assert c["steps"][10]["production"] == -0.0013657344567323075


def test_entropy_test_state_known_answers(port):
    for diss, tag in ((False, "ec"), (True, "diss")):
        k = K[f"entropy_test_20240501_{tag}"]
        s = port.mesh(po.bubble_mesh_config(1, True)).solver(4, "f64", settings=po.make_settings(diss))
        q = s.init_case(po.CASE_ENTROPY_TEST, 20240501).copy()
        assert np.array_equal(q, G["entropy_q"])
        rhs = s.assemble_rhs(q)
        assert np.array_equal(rhs, G[f"entropy_rhs_{tag}"])
        assert s.total_entropy(q) == k["entropy"] == -262277934766.46829
        assert s.entropy_production(q, rhs) == k["production"]
        # criterion 1 of the acceptance suite (acceptance.cpp:78-96)
        if not diss:
            assert abs(k["production"]) <= 1e-10 * abs(k["entropy"])
            assert k["production"] == -8.2658971223281696e-08
    assert np.array_equal(s.volume_rhs(q), G["entropy_volume_rhs"])


def test_fp32_golden(port):
    s = port.mesh(po.bubble_mesh_config(1, True)).solver(4, "f32")
    q = s.init_case(po.CASE_ENTROPY_TEST, 20240501).copy()
    assert np.array_equal(q, G["entropy_q_f32"])
    assert np.array_equal(s.assemble_rhs(q), G["entropy_rhs_diss_f32"])


def test_partitioned_trajectory_golden(port):
    """The reference's 2-rank run equals the serial oracle bitwise
    (test_partition.cpp:94-100)."""
    s = port.mesh(po.bubble_mesh_config(1, False)).solver(3, "f64")
    s.init_case(po.CASE_BUBBLE_SHARP)
    dt = s.compute_dt(0.5)
    assert dt == K["bubble_L1_N3"]["dt"]
    for _ in range(10):
        s.step(dt)
    assert np.array_equal(s.state, G["bubble_L1_N3_state10"])


def test_coriolis_golden(port):
    cfg = po.mesh_config((2, 1, 1), 1, (0., 0., 0.), (4e6, 6e6, 3e4), (0, 1, 1))
    s = port.mesh(cfg).solver(3, "f64", settings=po.make_settings(True, 2, 1e-4, 1.6e-11, 3e6))
    q = s.init_case(po.CASE_ENTROPY_TEST, 13).copy()
    assert np.array_equal(q, G["coriolis_q"])
    assert np.array_equal(s.assemble_rhs(q), G["coriolis_rhs"])


def test_rank_restricted_assembly_is_bitwise_serial(port):
    """The oracle's per-rank assembly with exchanged traces reproduces the
    serial result (solver.hpp:240-340 phase structure)."""
    mesh = port.mesh(po.bubble_mesh_config(1, True))
    s = mesh.solver(3, "f64")
    q = s.init_case(po.CASE_ENTROPY_TEST, 31).copy()
    serial = s.assemble_rhs(q)
    faces = mesh.faces
    for ranks in (2, 4):
        rb = port.partition(mesh.ne, ranks)
        out = np.zeros_like(q)
        for r in range(ranks):
            b, e = int(rb[r]), int(rb[r + 1])
            slot_of = -np.ones(mesh.nfaces, np.int32)
            traces = []
            for f, (me, pe, d, ms, refl) in enumerate(faces):
                if refl:
                    continue
                m_in, p_in = b <= me < e, b <= pe < e
                if m_in != p_in:
                    slot_of[f] = len(traces)
                    relem, rside = (pe, 1 - ms) if m_in else (me, ms)
                    traces.append(s.extract_trace(q, relem, d, rside))
            s.assemble_rhs_rank(q, out, 0.0, 1.0, b, e, slot_of, np.array(traces))
        assert np.array_equal(out, serial)


# ---- pointwise physics (reference tests/test_physics.cpp) -------------------

def _vals(s, rho, u, p, phi):
    q5 = np.array([rho, rho * u[0], rho * u[1], rho * u[2],
                   p / 0.4 + 0.5 * rho * sum(x * x for x in u) + rho * phi])
    rc, nv = s.node_vals(q5, phi)
    assert rc == 0
    return nv


@pytest.fixture(scope="module")
def pw(port):
    return port.mesh(po.unit_mesh_config(0)).solver(1, "f64")


def test_log_mean_limits(pw):
    """test_physics.cpp:70-92."""
    assert pw.log_mean(2.0, 2.0, math.log(2.0), math.log(2.0)) == 2.0
    got = pw.log_mean(1.0, 2.0, 0.0, math.log(2.0))
    assert abs(got - 1.0 / math.log(2.0)) <= 2e-16 * got
    a, b = 1.0, 1.0 + 1e-6   # series branch against a long series
    xi = (b - a) / (b + a)
    exact = 0.5 * (a + b) / (1 + xi ** 2 / 3 + xi ** 4 / 5 + xi ** 6 / 7)
    assert abs(pw.log_mean(a, b, math.log(a), math.log(b)) - exact) <= 2e-16 * exact


def test_spec_consistency_example(pw):
    """test_physics.cpp:139-150: F(q,q) = (2, 4+1e5, 0, 0, 2(2.5e5+2+1e5))."""
    v = _vals(pw, 1.0, (2.0, 0, 0), 1e5, 0.0)
    f = pw.ec_flux(v, v, 0)
    assert abs(f[0] - 2.0) <= 1e-13 * 2.0
    assert abs(f[1] - (4.0 + 1e5)) <= 1e-13 * 1e5
    assert f[2] == 0.0 and f[3] == 0.0 and f[5] == 0.0
    assert abs(f[4] - 2.0 * (2.5e5 + 2.0 + 1e5)) <= 1e-13 * 7e5
    assert [float(x) for x in f] == K["spec_consistency_flux"]


def test_rho_hat_gravity_example(pw):
    """test_physics.cpp:152-168: G = 1/2 rho_hat [[phi]] ~ 10.615."""
    m, p = _vals(pw, 1.0, (0, 0, 0), 1e5, 0.0), _vals(pw, 2.0, (0, 0, 0), 1e5, 9.81)
    f = pw.ec_flux(m, p, 0)
    assert abs(f[5] - 0.5 * 1.5 / math.log(2.0) * 9.81) <= 1e-12 * f[5]
    assert abs(f[5] - 10.615) <= 1e-3 * 10.615
    assert [float(x) for x in f] == K["rho_hat_example_flux"]
    # partner rule: -G b-/b+ equals the swapped evaluation
    g = pw.ec_flux(p, m, 0)
    assert abs(-f[5] * f[6] - g[5]) <= 1e-14 * abs(g[5])
    assert abs(g[5] + 5.3075) <= 1e-3 * 5.3075


def test_flux_consistency_and_symmetry_random(pw):
    """test_physics.cpp:112-137, 170-202 on seeded draws."""
    rng = np.random.default_rng(7)
    for _ in range(500):
        phi = rng.uniform(0, 2e4)
        rho, u, p = rng.uniform(0.5, 2.0), rng.uniform(-50, 50, 3), rng.uniform(5e4, 2e5)
        v = _vals(pw, rho, u, p, phi)
        E = p / 0.4 + 0.5 * rho * (u @ u) + rho * phi
        for d in range(3):
            f = pw.ec_flux(v, v, d)
            ana = np.array([rho * u[d], rho * u[0] * u[d], rho * u[1] * u[d], rho * u[2] * u[d], (E + p) * u[d]])
            ana[1 + d] += p
            assert np.all(np.abs(f[:5] - ana) <= 1e-13 * (np.abs(ana) + 1e-30))
            assert f[5] == 0.0
        w = _vals(pw, rng.uniform(0.5, 2.0), rng.uniform(-50, 50, 3), rng.uniform(5e4, 2e5), rng.uniform(0, 2e4))
        d = int(rng.integers(0, 3))
        f, g = pw.ec_flux(v, w, d), pw.ec_flux(w, v, d)
        assert np.array_equal(f[:5], g[:5])            # bitwise symmetric
        assert abs(-f[5] * f[6] - g[5]) <= 5e-16 * (abs(g[5]) + 1e-30)
        dm, dp = pw.matrix_dissipation(v, w, d), pw.matrix_dissipation(w, v, d)
        assert np.array_equal(dm, -dp)                 # antisymmetric under side swap
        assert np.all(pw.matrix_dissipation(v, v, d) == 0.0)   # test_physics.cpp:333-340


def test_pointwise_golden_pairs(pw):
    for row in G["pointwise_pairs"]:
        a8, b8, d = row[:8], row[8:16], int(row[16])
        assert np.array_equal(pw.ec_flux(a8, b8, d), row[17:24])
        assert np.array_equal(pw.matrix_dissipation(a8, b8, d), row[24:29])


def test_nonphysical_state(port):
    """test_kernels.cpp:279-288, error.hpp payload."""
    s = port.mesh(po.unit_mesh_config(1)).solver(2, "f64", gas=po.default_gas(0.0))
    q = s.init_case(po.CASE_CONSTANT, 0, [1.0, 0.0, 0.0, 0.0, 1e5]).copy()
    q[3, 0, 5] = -1.0
    with pytest.raises(po.NonPhysicalState) as e:
        s.assemble_rhs(q)
    assert (e.value.element, e.value.node, e.value.rho, e.value.pressure) == (3, 5, -1.0, 0.0)


def test_hydrostatic_and_free_stream(port):
    """test_kernels.cpp:30-44, 254-265."""
    s = port.mesh(po.bubble_mesh_config(1, False)).solver(4, "f64")
    rhs = s.assemble_rhs(s.init_case(po.CASE_HYDROSTATIC).copy())
    assert np.abs(rhs[:, 0]).max() == 0.0 and np.abs(rhs[:, 4]).max() == 0.0
    assert np.abs(rhs[:, 3]).max() > 0.0
    for order in (2, 3, 4):
        s = port.mesh(po.unit_mesh_config(1)).solver(order, "f64", gas=po.default_gas(0.0))
        rhs = s.assemble_rhs(s.init_case(po.CASE_CONSTANT, 0, [1.2, 20.0, 10.0, 5.0, 1e5]).copy())
        assert np.abs(rhs).max() <= 1e-13 * (2.0 * 4.0 * 10.0 * 1e5)


def test_lsrk_order_four(port):
    """test_time_integration.cpp:34-60 in spirit: halving dt on a smooth
    state reduces the one-step-pair difference by ~2^4 (observed order)."""
    cfg = po.bubble_mesh_config(1, True)
    errs = []
    T = 0.4
    ref_state = None
    for n in (16, 8, 4, 2):
        s = port.mesh(cfg).solver(3, "f64", settings=po.make_settings(False))
        s.init_case(po.CASE_ENTROPY_TEST, 3)
        for _ in range(n):
            s.step(T / n)
        if ref_state is None:
            ref_state = s.state.copy()
        else:
            errs.append(float(np.abs(s.state - ref_state).max()))
    rate = math.log2(errs[2] / errs[1])
    assert 3.5 <= rate <= 5.2, (errs, rate)


def test_sampled_assembly_equals_full_assembly(port):
    """The machinery of tests/test_gpu_stage_parity.py's bench-size check:
    assemble_rhs_rank on element ranges with the neighbours' traces taken from
    the full state reproduces the full assembly bitwise on those elements, and
    flux_scale_rank over ranges that cover the mesh gives flux_scale."""
    from helpers import check_samples, face_table, sample_ranges
    for periodic in (False, True):
        omesh = port.mesh(po.bubble_mesh_config(2, periodic))
        o = omesh.solver(3, "f64")
        q = o.init_case(po.CASE_ENTROPY_TEST, 8).copy()
        full = o.assemble_rhs(q)
        rng = np.random.default_rng(1)
        ranges = sample_ranges(omesh.ne, 5, 4, rng)
        worst, n = check_samples(o, omesh.face_of, face_table(omesh), q, full, ranges, 0.0)
        assert worst == 0.0 and n >= 100
        slot = np.full(omesh.nfaces, -1, np.int32)
        whole = o.flux_scale_rank(q, 0, omesh.ne, slot, np.zeros((1, 5, 16)))
        assert np.array_equal(whole, o.flux_scale(q))
