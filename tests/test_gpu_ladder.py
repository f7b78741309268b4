"""The optimisation ladder of the volume kernel as run-time selectable GPU
kernels (-m gpu): KernelSettings::variant (kernels.hpp:27-34) -> one volume
kernel per rung (baseline/fused, precompute, logmean, symmetric/balanced; see
dev::kRung* in csrc/esdg_device.cuh).

The reference gates its ladder on equivalence: every variant must reproduce the
balanced tendency (ladder.hpp:28-58, tests/test_kernels.cpp:69-93, 1e-13 of
max|rhs| on its well-conditioned state). Here every rung is compared with the
oracle's (balanced) volume_rhs at the tolerance of the product kernel, and the
reference's own max_rel_diff is reported alongside.
"""
import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2605_16684_b200 import capi
from helpers import max_rel_diff, scaled_error
from test_gpu_parity import TOL32, TOL64, make

pytestmark = pytest.mark.gpu

VARIANTS = ["baseline", "fused", "precompute", "logmean", "symmetric", "balanced"]


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("order", [2, 4, 5])
@pytest.mark.parametrize("variant", range(6), ids=VARIANTS)
def test_every_rung_matches_the_oracle(port, variant, order, prec):
    o, g = make(port, "bubble", (1, True), order, prec=prec)
    q = o.init_case(po.CASE_ENTROPY_TEST, 20240501).copy()
    want = o.volume_rhs(q)
    scale = o.flux_scale(q)
    g.set_variant(variant)
    got = g.volume_rhs(q)
    tol = TOL64 if prec == "f64" else TOL32
    assert scaled_error(got, want, scale) <= tol
    # ladder.hpp:14-22; the reference's gate is 1e-13 between its own variants
    # (identical arithmetic up to summation order); GPU vs CPU keeps the level
    # of the product kernel
    assert max_rel_diff(got, want) <= (2e-11 if prec == "f64" else 2e-4)


@pytest.mark.parametrize("path", [capi.PATH_SPLIT, capi.PATH_STAGE])
@pytest.mark.parametrize("variant", [0, 2, 3], ids=["baseline", "precompute", "logmean"])
def test_rung_in_the_full_rhs(port, variant, path):
    """assemble_rhs with a rung below "symmetric" selected: the split structure
    (ladder volume kernel + surface kernel) serves it on every path, walls and
    periodic faces, two partitions."""
    o, g = make(port, "bubble", (2, False), 4, ranks=2, path=path)
    q = o.init_case(po.CASE_ENTROPY_TEST, 99).copy()
    g.set_variant(variant)
    assert scaled_error(g.assemble_rhs(q), o.assemble_rhs(q), o.flux_scale(q)) <= TOL64
    g.set_variant(5)
    assert scaled_error(g.assemble_rhs(q), o.assemble_rhs(q), o.flux_scale(q)) <= TOL64


def test_rungs_agree_with_each_other(port):
    """The reference's own gate (test_kernels.cpp:69-93): all variants within
    1e-13 of the balanced one. The two division formulations differ by an ulp
    per quotient, so the GPU rungs keep 1e-12 of the flux scale among
    themselves."""
    o, g = make(port, "bubble", (1, True), 4)
    q = o.init_case(po.CASE_ENTROPY_TEST, 7).copy()
    scale = o.flux_scale(q)
    g.set_variant(5)
    ref = g.volume_rhs(q)
    for v in range(5):
        g.set_variant(v)
        assert scaled_error(g.volume_rhs(q), ref, scale) <= 1e-12, VARIANTS[v]
