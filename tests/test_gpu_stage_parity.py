"""Oracle parity of the path bench.py times by default (-m gpu): the
one-kernel-per-stage path (PATH_STAGE, rhs_kernel<...,VOL,SURF> with the fused
LSRK update) at every order and precision, with walls and periodic boundaries,
on one and three partitions -- and at the size bench.py runs (BASELINE.json
configs[1], 884,736 elements), where the oracle is evaluated on sampled
elements only.

The orders take different code: TMA slab commit for odd NQ, per-thread commit
for even NQ (N = 1, 3, 5, 7), the lean line state at N = 6, 7, the flat x/y
sweep at N = 6, paired faces per iteration at N = 3 and N >= 5.

Tolerances as in test_gpu_parity.py: FP64 RHS 2e-12 of the abs-sum flux scale
(typical 1e-13 .. 7e-13; 1.41e-12 once in 680 random trials, pinned below),
FP32 3e-5; five-step states 1e-11 / 1e-4 of max|q_v| (measured 2e-12 / 2e-5).
"""
import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2605_16684_b200 import capi
from helpers import (both_configs, check_samples, face_table, gas_pair, sample_ranges, scaled_error,
                     settings_pair, state_error)
from test_gpu_parity import TOL32, TOL64, make

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ranks", [1, 3])
@pytest.mark.parametrize("periodic", [False, True], ids=["walls", "periodic"])
@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("order", [1, 2, 3, 4, 5, 6, 7])
def test_stage_path_rhs_and_trajectory(port, order, prec, periodic, ranks):
    """RHS through rhs() (the stage kernel without the update) and five LSRK
    steps through the stage kernel against the oracle's assemble_rhs / step.
    64 elements: several CTAs at every order, partitions of 21-22 elements
    whose element groups straddle partition boundaries."""
    level = 2 if order <= 5 else 1
    o, g = make(port, "bubble", (level, periodic), order, prec=prec, ranks=ranks, path=capi.PATH_STAGE)
    q = o.init_case(po.CASE_ENTROPY_TEST, 1000 + 10 * order + ranks).copy()
    scale = o.flux_scale(q)
    tol_rhs, tol_q = (TOL64, 1e-11) if prec == "f64" else (TOL32, 1e-4)
    want, got = o.assemble_rhs(q), g.assemble_rhs(q)
    assert scaled_error(got, want, scale) <= tol_rhs
    # accumulate form with the stage coefficients' signs (a_old < 0)
    out0 = (np.random.default_rng(order).standard_normal(q.shape) * scale[None, :, None]).astype(q.dtype)
    want = o.assemble_rhs(q, out0.copy(), -0.4178904745, 0.5)
    got = g.assemble_rhs(q, out0.copy(), -0.4178904745, 0.5)
    assert scaled_error(got, want, scale) <= tol_rhs
    o.state[:] = q
    g.set_state(q)
    dt = o.compute_dt(0.4)
    dt = float(np.float32(dt)) if prec == "f32" else dt
    for _ in range(5):
        o.step(dt)
        g.step(dt)
    gs = g.get_state()
    err = state_error(gs, o.state)
    assert err[0] <= tol_q and err[4] <= tol_q, err
    mom = float(np.abs(o.state[:, 1:4]).max())
    assert float(np.abs(gs[:, 1:4].astype(np.float64) - o.state[:, 1:4]).max()) <= 10 * tol_q * mom
    # the k register the stage kernel leaves behind is the oracle's too: five
    # steps of state differences (tol_q of max|q|) feed back into it, so it is
    # compared at that level of the flux scale (measured 1.5e-3 FP32 worst)
    k_scale = dt * scale + 1e-300
    assert scaled_error(g.get_state(capi.REG_K), o.kreg, k_scale) <= 50 * tol_q


@pytest.mark.parametrize("path", [capi.PATH_SPLIT, capi.PATH_FUSED, capi.PATH_STAGE])
@pytest.mark.parametrize("ranks", [1, 4])
def test_fuzz_outlier_regression(port, path, ranks):
    """The one trial of 680 randomised comparisons (tools/fuzz_parity.py seed 0,
    trial 138; profiles/r1_fuzz_parity.txt) above the survey's 1e-12: N = 6,
    walls, no dissipation, EntropyTestState seed 603644430. The energy
    tendency differs by 1.41e-12 of its flux scale, every other variable by
    <= 5e-16, for every a_new, path and partition count: a logarithmic mean next
    to its series threshold xi^2 = 1e-8, where the device logarithm (0.53 ulp)
    and glibc's (< 1 ulp) may differ by an ulp that the quotient amplifies by
    1/(2 xi) = 5e3. This is why the stated FP64 bound is 2e-12 and not 1e-12;
    the test pins the level so a regression of the logarithm or of the branch
    selector shows up."""
    o, g = make(port, "bubble", (1, False), 6, diss=False, ranks=ranks, path=path)
    q = o.init_case(po.CASE_ENTROPY_TEST, 603644430).copy()
    scale = o.flux_scale(q)
    want, got = o.assemble_rhs(q), g.assemble_rhs(q)
    per = [float(np.abs(got[:, v] - want[:, v]).max()) / scale[v] for v in range(5)]
    assert max(per[:4]) <= 1e-14, per
    assert per[4] <= 1.6e-12, per


@pytest.mark.parametrize("path", [capi.PATH_SPLIT, capi.PATH_STAGE])
@pytest.mark.parametrize("ranks", [1, 2])
def test_fuzz_outlier_regression_second(port, path, ranks):
    """The worst of 2,160 further randomised comparisons at the end of round 2
    (tools/fuzz_parity.py seed 108, trial 49; profiles/r2_fuzz_parity_seed2.txt):
    N = 4, walls, dissipation on, 64 elements, EntropyTestState seed 193596780.
    Same signature as the first outlier: the energy tendency of one node
    (element 26, node 2) differs by 1.72e-12 of its flux scale, mass by 7e-15,
    the momenta by 2e-16, for every a_new, path and partition count
    (tools/fuzz_replay.py 108 49) -- a logarithmic mean of b next to its series
    threshold. Pinned at its level, inside the stated 2e-12."""
    o, g = make(port, "bubble", (2, False), 4, diss=True, ranks=ranks, path=path)
    q = o.init_case(po.CASE_ENTROPY_TEST, 193596780).copy()
    scale = o.flux_scale(q)
    want, got = o.assemble_rhs(q), g.assemble_rhs(q)
    per = [float(np.abs(got[:, v] - want[:, v]).max()) / scale[v] for v in range(5)]
    assert max(per[:4]) <= 5e-14, per
    assert per[4] <= 1.9e-12, per


def test_rhs_against_unmodified_reference(ref, port):
    """The GPU RHS compared DIRECTLY with the unmodified reference
    (oracle/_ref/libesdg_ref.so, which travels to the GPU box prebuilt), not
    only transitively through the restatement."""
    for order, prec, tol in ((4, "f64", TOL64), (5, "f64", TOL64), (4, "f32", TOL32)):
        oc, cc = both_configs("bubble", 1, True)
        r = ref.mesh(oc).solver(order, prec)
        p = port.mesh(oc).solver(order, prec)
        g = capi.GpuSolver(capi.Mesh(cc), order, prec)
        g.set_path(capi.PATH_STAGE)
        q = r.init_case(po.CASE_ENTROPY_TEST, 20240501).copy()
        want, got = r.assemble_rhs(q), g.assemble_rhs(q)
        assert scaled_error(got, want, p.flux_scale(q)) <= tol


# ---- bench size ---------------------------------------------------------------

def test_bench_size_sampled_parity(port):
    """BASELINE.json configs[1] as bench.py runs it: N = 4, base 3^3 at
    refinement 5 = 884,736 elements (176,948 CTAs, ~400 resident waves, L2
    prefetch distance logic, a last CTA with one element). One assemble_rhs on
    the GPU; the oracle evaluates ~190 sampled elements (assemble_rhs_rank with
    the neighbours' traces taken from the full state): first / last CTA, both
    sides of the step_swap run boundaries and random places. Then one
    step_swap (the call bench.py's e2e arm times) against step + get_state,
    bitwise."""
    cfg_o = po.bubble_mesh_config(5, False, base=(3, 3, 3))
    cfg_g = capi.bubble_mesh_config(5, False, base=(3, 3, 3))
    g = capi.GpuSolver(capi.Mesh(cfg_g), 4, "f64")
    g.set_path(capi.PATH_STAGE)
    g.init_case(capi.CASE_BUBBLE_SHARP)
    q = g.get_state()
    assert q.shape == (884736, 5, 125)
    # a rough state on top of the bubble so that every term is exercised:
    # smooth, deterministic, 1e-3 relative
    rng = np.random.default_rng(5)
    q *= 1.0 + 1e-3 * np.sin(np.arange(q.shape[0], dtype=np.float64) * 0.37)[:, None, None]
    q[:, 1:4] += 0.5 * rng.standard_normal((q.shape[0], 3, 1))
    got = g.assemble_rhs(q)
    omesh = port.mesh(cfg_o)
    o = omesh.solver(4, "f64")
    faces, face_of = face_table(omesh), omesh.face_of
    ranges = sample_ranges(q.shape[0], 5, 8, rng)
    worst, n = check_samples(o, face_of, faces, q, got, ranges, TOL64)
    print(f"bench-size parity: {n} sampled elements, scaled error {worst:.2e}")
    # step_swap at this size: eight runs of the last stage leaving for the host
    g.set_state(q)
    dt = 0.5 * g.compute_dt(0.5)
    out = g.step_swap(dt, q)
    g2 = capi.GpuSolver(capi.Mesh(cfg_g), 4, "f64")
    g2.set_path(capi.PATH_STAGE)
    g2.set_state(q)
    g2.step(dt)
    assert np.array_equal(out, g2.get_state())


# the other points of the configs[1] order / precision sweep at the sizes
# tools/sweep_probe.py and bench.py --order run them (~1e8 DOF each)
SWEEP_POINTS = [(5, (5, 5, 5), 4, "f64"), (6, (1, 1, 1), 6, "f64"), (7, (15, 15, 15), 2, "f64"),
                (4, (3, 3, 3), 5, "f32"), (5, (5, 5, 5), 4, "f32"), (6, (1, 1, 1), 6, "f32"),
                (7, (15, 15, 15), 2, "f32")]


@pytest.mark.parametrize("order,base,refinement,prec", SWEEP_POINTS,
                         ids=[f"N{p[0]}-{p[3]}" for p in SWEEP_POINTS])
def test_sweep_size_sampled_parity(port, order, base, refinement, prec):
    """The order / precision sweep of BASELINE.json configs[1] at its own sizes
    (N = 5, 6, 7 in FP64, N = 4 ... 7 in FP32; ~1e8 DOF each): one assemble_rhs
    on the stage path, the oracle on ~190 sampled elements (first / last element
    group, evenly spaced group boundaries, random places), as
    test_bench_size_sampled_parity does for N = 4 FP64."""
    cfg_o = po.bubble_mesh_config(refinement, False, base=base)
    cfg_g = capi.bubble_mesh_config(refinement, False, base=base)
    g = capi.GpuSolver(capi.Mesh(cfg_g), order, prec)
    g.set_path(capi.PATH_STAGE)
    g.init_case(capi.CASE_BUBBLE_SHARP)
    q = g.get_state()
    ne = q.shape[0]
    assert ne == base[0] * base[1] * base[2] * 8 ** refinement and 8.5e7 < q.size / 5 < 1.2e8
    rng = np.random.default_rng(order)
    q *= (1.0 + 1e-3 * np.sin(np.arange(ne, dtype=np.float64) * 0.37)).astype(q.dtype)[:, None, None]
    q[:, 1:4] += (0.5 * rng.standard_normal((ne, 3, 1))).astype(q.dtype)
    got = g.assemble_rhs(q)
    omesh = port.mesh(cfg_o)
    o = omesh.solver(order, prec)
    faces, face_of = face_table(omesh), omesh.face_of
    # elements per CTA differ by order and precision (1 .. 10): 5 and 7 give
    # group boundaries of both kinds
    ranges = sample_ranges(ne, 5, 8, rng) + sample_ranges(ne, 7, 4, rng)[:6]
    if prec == "f64":
        worst, n = check_samples(o, face_of, faces, q, got, ranges, TOL64)
        print(f"sweep-size parity N={order} f64: {n} sampled elements, scaled error {worst:.2e}")
        return
    # FP32 at 1e8 DOF: neighbouring nodes of so fine a mesh are so close that the
    # logarithmic means sit next to their series threshold, where the difference
    # of two FP32 logarithms (|log b| = 11.5, one ulp 9.5e-7) carries 1e-4 ... 1e-3
    # of relative error in the reference's FP32 build and here alike (DESIGN.md
    # section 6). The FP64 oracle is the judge of both: the GPU FP32 result must be
    # as close to it as the FP32 oracle is (factor 1.5), and the three distances
    # are printed.
    o64 = omesh.solver(order, "f64")
    q64 = q.astype(np.float64)
    inf = float("inf")
    d_gpu, n = check_samples(o64, face_of, faces, q64, got.astype(np.float64), ranges, inf)
    g64 = capi.GpuSolver(capi.Mesh(cfg_g), order, "f64")
    g64.set_path(capi.PATH_STAGE)
    truth = g64.assemble_rhs(q64)
    d_truth, _ = check_samples(o64, face_of, faces, q64, truth, ranges, TOL64)
    d_or32, _ = check_samples(o, face_of, faces, q, truth.astype(np.float32), ranges, inf)
    d_pair, _ = check_samples(o, face_of, faces, q, got, ranges, inf)
    print(f"sweep-size parity N={order} f32: {n} sampled elements; of the flux scale: GPU f32 vs f64 oracle "
          f"{d_gpu:.2e}, f32 oracle vs f64 {d_or32:.2e}, GPU f32 vs f32 oracle {d_pair:.2e} "
          f"(GPU f64 vs f64 oracle {d_truth:.2e})")
    assert d_gpu <= max(TOL32, 1.5 * d_or32)


def test_channel_size_sampled_parity(port):
    """BASELINE.json configs[2] as bench.py --case baroclinic runs it: channel
    mesh (12, 2, 1) at refinement 5 = 786,432 elements, N = 4 FP64 (98.3 MDOF),
    beta-plane Coriolis, dissipation on, walls in y and z, periodic in x; the
    perturbed balanced jet plus a rough 1e-3 modulation. One assemble_rhs on
    the stage path; the oracle (same Coriolis settings) on sampled elements."""
    cor = (2, 1e-4, 1.6e-11, 3e6)
    margs = ((12, 2, 1), 5, (0., 0., 0.), (4e7, 6e6, 3e4), (0, 1, 1))
    oc, cc = both_configs("raw", *margs)
    so, sc = settings_pair(True, *cor)
    go, gc = gas_pair(9.81)
    g = capi.GpuSolver(capi.Mesh(cc), 4, "f64", gas=gc, settings=sc)
    g.set_path(capi.PATH_STAGE)
    g.init_case(capi.CASE_BAROCLINIC_JET)
    q = g.get_state()
    ne = q.shape[0]
    assert ne == 786432 and float(np.abs(q[:, 1] / q[:, 0]).max()) > 25.0   # there is a jet
    rng = np.random.default_rng(17)
    q *= 1.0 + 1e-3 * np.sin(np.arange(ne, dtype=np.float64) * 0.37)[:, None, None]
    q[:, 2:4] += 0.05 * rng.standard_normal((ne, 2, 1))
    got = g.assemble_rhs(q)
    omesh = port.mesh(oc)
    o = omesh.solver(4, "f64", gas=go, settings=so)
    faces, face_of = face_table(omesh), omesh.face_of
    ranges = sample_ranges(ne, 5, 8, rng)
    worst, n = check_samples(o, face_of, faces, q, got, ranges, TOL64)
    print(f"channel-size parity: {n} sampled elements, scaled error {worst:.2e}")


def test_bench_size_partition_bitwise():
    """Size-independent property at configs[1] itself (884,736 elements): the
    state after one LSRK step on four Morton ranges (packed traces, interior /
    boundary element groups, ghost faces evaluated by both sides) equals the
    one-partition result bit for bit, on the stage path bench.py times
    (tests/test_partition.cpp:94-114 at the bench size)."""
    cfg = capi.bubble_mesh_config(5, False, base=(3, 3, 3))
    states = []
    for ranks in (1, 4):
        g = capi.GpuSolver(capi.Mesh(cfg), 4, "f64", ranks=ranks)
        g.set_path(capi.PATH_STAGE)
        g.init_case(capi.CASE_BUBBLE_SHARP)
        if ranks == 1:
            dt = 0.5 * g.compute_dt(0.5)
        g.step(dt)
        states.append(g.get_state())
        del g
    assert np.isfinite(states[0]).all()
    assert np.array_equal(states[0], states[1])


def test_bench_size_conservation_properties():
    """Size-independent properties at the size of configs[1] (884,736
    elements), evaluated by the device reductions (K6) on the k register of one
    stage-path RHS of a rough state: mass and energy rates vanish; on the
    periodic copy of the mesh with the dissipation off so does the entropy
    production (test_kernels.cpp:164-183, 202-252; acceptance 1-2); on the mesh
    as benched (walls) with the matrix dissipation on the production is
    negative. (Dissipation on a mesh that is periodic in the direction of
    gravity does not conserve energy, in the reference as here: phi jumps across
    the wrap.)"""
    prod = {}
    for diss, periodic in ((0, True), (1, False)):
        cfg = capi.bubble_mesh_config(5, periodic, base=(3, 3, 3))
        g = capi.GpuSolver(capi.Mesh(cfg), 4, "f64", settings=capi.Settings(diss, 0, 0.0, 0.0, 0.0))
        g.set_path(capi.PATH_STAGE)
        g.init_case(capi.CASE_BUBBLE_SHARP)
        q = g.get_state()
        ne = q.shape[0]
        rng = np.random.default_rng(3)
        q *= 1.0 + 1e-3 * np.sin(np.arange(ne, dtype=np.float64) * 0.37)[:, None, None]
        q[:, 1:4] += 0.5 * rng.standard_normal((ne, 3, 1))
        g.set_state(q)
        dt = g.compute_dt(0.5)
        mass, energy, eta = g.quadrature_total(0), g.quadrature_total(4), g.total_entropy()
        g.rhs(0.0, 1.0)
        rates = g.quadrature_total(0, capi.REG_K), g.quadrature_total(4, capi.REG_K)
        prod[diss] = g.entropy_production()
        print(f"bench-size conservation (dissipation {diss}): mass drift per step {rates[0] * dt / mass:.2e}, "
              f"energy {rates[1] * dt / energy:.2e}, entropy production {prod[diss]:.3e} (eta {eta:.3e})")
        assert abs(rates[0]) * dt <= 1e-13 * abs(mass)
        assert abs(rates[1]) * dt <= 1e-13 * abs(energy)
        del g
    assert abs(prod[0]) <= 1e-10 * abs(eta)
    assert prod[1] < 0.0 and abs(prod[1]) > 1e3 * abs(prod[0])


def test_bench_size_step_stream_bitwise():
    """The call bench.py's e2e figure times, at its size: two independent
    states of configs[1] streamed through one solver (upload of the next and
    download of the previous beside the step) equal set_state + step +
    get_state per member, bit for bit."""
    cfg = capi.bubble_mesh_config(5, False, base=(3, 3, 3))
    g = capi.GpuSolver(capi.Mesh(cfg), 4, "f64")
    g.set_path(capi.PATH_STAGE)
    g.init_case(capi.CASE_BUBBLE_SHARP)
    a = g.get_state()
    b = a * (1.0 + 1e-3 * np.cos(np.arange(a.shape[0], dtype=np.float64) * 0.11))[:, None, None]
    dt = 0.5 * g.compute_dt(0.5)
    want = []
    for q in (a, b):
        g.set_state(q)
        g.step(dt)
        want.append(g.get_state())
    out_a = np.empty_like(a)
    g.set_state(a)
    g.step_stream(dt, b, None)        # steps a, uploads b
    g.step_stream(dt, None, out_a)    # steps b, downloads a's result
    assert np.array_equal(out_a, want[0])
    assert np.array_equal(g.get_state(), want[1])
    assert not np.array_equal(want[0], want[1])
