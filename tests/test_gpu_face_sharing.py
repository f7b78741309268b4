"""Shared face evaluation of the one-pass kernels (-m gpu).

PATH_FUSED / PATH_STAGE evaluate every interior face once: the element on the
minus side works out both elements' lift terms and hands the other one its
share through device memory (RhsParams::face_roles, esdg_kernels.cuh), the way
the reference keeps ONE record per face that commit_face_side reads for both
sides (kernels.hpp:350-430). The handed-over number is bitwise what the
receiving element computes when it evaluates the face itself, so

  * sharing on == sharing off, bitwise, for the RHS and for trajectories;
  * the result does not depend on the partition count (a face that is local in
    one partitioning is a ghost face, evaluated by both ranks, in another) --
    tests/test_partition.cpp:94-114 of the reference;
  * launches over lists (interior / boundary groups) and over consecutive runs
    of groups (step_swap) agree with one launch over everything.
"""
import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2605_16684_b200 import capi
from helpers import both_configs, scaled_error
from test_gpu_parity import TOL32, TOL64, make

pytestmark = pytest.mark.gpu


def solver(cfg, order, prec, path, ranks=1, share=True, diss=True, overlap=True):
    g = capi.GpuSolver(capi.Mesh(cfg), order, prec, settings=capi.Settings(int(diss), 0, 0.0, 0.0, 0.0),
                       ranks=ranks)
    g.set_path(path)
    g.set_face_sharing(share)
    g.set_overlap(overlap)
    return g


@pytest.mark.parametrize("path", [capi.PATH_FUSED, capi.PATH_STAGE])
@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("order", [1, 2, 3, 4, 5, 6, 7])
def test_sharing_is_bitwise_neutral(port, order, prec, path):
    """RHS (overwrite and accumulate form) and three LSRK steps with the faces
    shared against every element evaluating its own six, on a mesh with walls
    AND periodic wrap-around (so all three kinds of - faces occur: pulled,
    wall, wrap-around evaluated in place)."""
    level = 2 if order <= 5 else 1
    oc, cc = both_configs("bubble", level, False)
    o = port.mesh(oc).solver(order, prec)
    q = o.init_case(po.CASE_ENTROPY_TEST, 77 + order).copy()
    a, b = solver(cc, order, prec, path, share=True), solver(cc, order, prec, path, share=False)
    ra, rb = a.assemble_rhs(q), b.assemble_rhs(q)
    assert np.array_equal(ra, rb)
    # and it is the right answer
    assert scaled_error(ra, o.assemble_rhs(q), o.flux_scale(q)) <= (TOL64 if prec == "f64" else TOL32)
    out0 = np.random.default_rng(order).standard_normal(q.shape).astype(q.dtype)
    assert np.array_equal(a.assemble_rhs(q, out0.copy(), -0.4178904745, 0.5),
                          b.assemble_rhs(q, out0.copy(), -0.4178904745, 0.5))
    dt = o.compute_dt(0.4)
    dt = float(np.float32(dt)) if prec == "f32" else dt
    for g in (a, b):
        g.set_state(q)
        for _ in range(3):
            g.step(dt)
    assert np.array_equal(a.get_state(), b.get_state())
    assert np.array_equal(a.get_state(capi.REG_K), b.get_state(capi.REG_K))


@pytest.mark.parametrize("path", [capi.PATH_FUSED, capi.PATH_STAGE])
@pytest.mark.parametrize("periodic", [False, True], ids=["walls", "periodic"])
def test_sharing_partition_independent(port, path, periodic):
    """1 / 2 / 3 / 8 partitions, overlap on and off (list launches and one
    launch), shared faces: bitwise one result."""
    oc, cc = both_configs("bubble", 2, periodic)
    o = port.mesh(oc).solver(4, "f64")
    q = o.init_case(po.CASE_ENTROPY_TEST, 4242).copy()
    dt = o.compute_dt(0.4)
    ref_rhs = ref_q = None
    for ranks in (1, 2, 3, 8):
        for overlap in (True, False):
            g = solver(cc, 4, "f64", path, ranks=ranks, overlap=overlap)
            rhs = g.assemble_rhs(q)
            g.set_state(q)
            for _ in range(2):
                g.step(dt)
            qq = g.get_state()
            if ref_rhs is None:
                ref_rhs, ref_q = rhs, qq
            assert np.array_equal(rhs, ref_rhs), (ranks, overlap)
            assert np.array_equal(qq, ref_q), (ranks, overlap)


def test_sharing_without_dissipation_and_with_coriolis(port):
    """EC flux only (the dissipation's exact zeros must not pick up a sign) and
    the beta-plane source on a channel mesh with walls in y and z."""
    oc, cc = both_configs("bubble", 2, True)
    o = port.mesh(oc).solver(3, "f64")
    q = o.init_case(po.CASE_ENTROPY_TEST, 5).copy()
    a = solver(cc, 3, "f64", capi.PATH_STAGE, share=True, diss=False)
    b = solver(cc, 3, "f64", capi.PATH_STAGE, share=False, diss=False)
    ra, rb = a.assemble_rhs(q), b.assemble_rhs(q)
    assert ra.tobytes() == rb.tobytes()


def test_step_swap_runs_share_faces(port):
    """step_swap issues the last stage as consecutive runs of element groups;
    an element of one run pulls from elements of the runs before it. Against
    step + get_state, bitwise, with sharing on and off."""
    oc, cc = both_configs("bubble", 3, False)
    o = port.mesh(oc).solver(4, "f64")
    q = o.init_case(po.CASE_ENTROPY_TEST, 31).copy()
    dt = 0.5 * o.compute_dt(0.5)
    outs = []
    for share in (True, False):
        g = solver(cc, 4, "f64", capi.PATH_STAGE, share=share)
        g.set_state(q)
        outs.append(g.step_swap(dt, q))
        g2 = solver(cc, 4, "f64", capi.PATH_STAGE, share=share)
        g2.set_state(q)
        g2.step(dt)
        assert np.array_equal(outs[-1], g2.get_state())
    assert np.array_equal(outs[0], outs[1])
