"""esdg_b200_solver_step_stream (-m gpu): independent states streamed through
one solver -- while a member of an ensemble is stepped on the device, the next
member's state is uploaded and the previous member's result is downloaded.

The call bench.py's e2e arm times. What it must guarantee:

  * every member's trajectory is BITWISE the one esdg_b200_solver_step produces
    for that member alone (Solver::step, solver.hpp:132-146), and agrees with
    the oracle's Solver::step to the tests' tolerance;
  * the k register and the device state after the last call are those of the
    plain sequence;
  * the parked-result protocol is enforced (a parked result must be collected,
    none can be asked for when there is none), on every path and partition
    count;
  * a non-physical member is reported by the call that stepped it.
"""
import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2605_16684_b200 import capi
from helpers import both_configs
from test_gpu_parity import make

pytestmark = pytest.mark.gpu


def members_of(o, n=3):
    return [o.init_case(po.CASE_ENTROPY_TEST, 31 + 7 * m).copy() for m in range(n)]


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("order", [2, 3, 4, 5, 7])
def test_ensemble_round_robin_is_bitwise_step(port, order, prec):
    """Three members, three rounds, the loop of bench.py: call i steps member
    i mod 3, uploads member (i+1) mod 3 and downloads the result of member
    (i-1) mod 3 into that member's host buffer."""
    level = 2 if order <= 4 else 1
    oc, _ = both_configs("bubble", level, False)
    o = port.mesh(oc).solver(order, prec)
    start = members_of(o)
    dt = 2.0 ** -10   # exact in FP32 as well
    rounds = 3

    # the plain sequence, one member at a time
    _, g = make(port, "bubble", (level, False), order, prec=prec, path=capi.PATH_STAGE)
    want = []
    for q in start:
        g.set_state(q)
        traj = []
        for _ in range(rounds):
            g.step(dt)
            traj.append(g.get_state().copy())
        want.append(traj)
    want_k = g.get_state(capi.REG_K).copy()  # member 2's last step

    # and it is the right answer (first step of member 0 against the oracle)
    o.state[...] = start[0]
    o.step(dt)
    scale = np.abs(start[0]).max(axis=(0, 2), keepdims=True).astype(np.float64)
    assert np.max(np.abs(want[0][0].astype(np.float64) - np.asarray(o.state, np.float64)) / scale) <= (
        1e-12 if prec == "f64" else 1e-5)

    # streamed
    _, s = make(port, "bubble", (level, False), order, prec=prec, path=capi.PATH_STAGE)
    host = [q.copy() for q in start]
    seen = [[] for _ in start]
    s.set_state(host[0])
    n_calls = 3 * rounds
    for i in range(n_calls):
        last = i == n_calls - 1
        prev = (i + 2) % 3
        s.step_stream(dt, None if last else host[(i + 1) % 3], host[prev] if i > 0 else None)
        if i > 0:
            seen[prev].append(host[prev].copy())
    # the last call had no next state: its result is REG_Q, nothing is parked
    seen[(n_calls - 1) % 3].append(s.get_state().copy())
    with pytest.raises(capi.EsdgError):
        s.stream_collect()
    for m in range(3):
        assert len(seen[m]) == rounds
        for a, b in zip(seen[m], want[m]):
            assert np.array_equal(a, b)
    assert np.array_equal(s.get_state(capi.REG_K), want_k)


def test_collect_and_protocol(port):
    oc, _ = both_configs("bubble", 1, False)
    o = port.mesh(oc).solver(3, "f64")
    a, b = members_of(o, 2)
    _, g = make(port, "bubble", (1, False), 3, path=capi.PATH_STAGE)
    g.set_state(a)
    g.step(2e-3)
    want_a = g.get_state().copy()
    g.set_state(b)
    g.step(2e-3)
    want_b = g.get_state().copy()

    _, s = make(port, "bubble", (1, False), 3, path=capi.PATH_STAGE)
    s.set_state(a)
    out = np.empty_like(a)
    with pytest.raises(capi.EsdgError):      # nothing parked yet
        s.step_stream(2e-3, b, out)
    s.step_stream(2e-3, b, None)             # a's result is parked, b is the state
    assert np.array_equal(s.get_state(), b)
    with pytest.raises(capi.EsdgError):      # the parked result must be taken
        s.step_stream(2e-3, None, None)
    assert np.array_equal(s.stream_collect(), want_a)
    s.step(2e-3)                             # plain calls go on working on REG_Q
    assert np.array_equal(s.get_state(), want_b)


@pytest.mark.parametrize("ranks,path", [(2, capi.PATH_STAGE), (3, capi.PATH_STAGE), (1, capi.PATH_SPLIT),
                                        (2, capi.PATH_SPLIT), (1, capi.PATH_FUSED), (4, capi.PATH_FUSED)])
def test_every_path_and_partition_count(port, ranks, path):
    """Several partitions on the device (their halo exchange runs on its own
    copy stream while the state transfers use theirs) and the paths whose
    update is a separate kernel: three members, two rounds, bitwise step()."""
    oc, _ = both_configs("bubble", 2, False)
    o = port.mesh(oc).solver(3, "f64")
    start = members_of(o)
    dt, rounds = 1e-3, 2
    _, g = make(port, "bubble", (2, False), 3, ranks=ranks, path=path)
    want = []
    for q in start:
        g.set_state(q)
        for _ in range(rounds):
            g.step(dt)
        want.append(g.get_state().copy())
    _, s = make(port, "bubble", (2, False), 3, ranks=ranks, path=path)
    host = [q.copy() for q in start]
    s.set_state(host[0])
    n_calls = 3 * rounds
    for i in range(n_calls):
        s.step_stream(dt, None if i == n_calls - 1 else host[(i + 1) % 3], host[(i + 2) % 3] if i > 0 else None)
    assert np.array_equal(host[0], want[0]) and np.array_equal(host[1], want[1])
    assert np.array_equal(s.get_state(), want[2])


def test_nonphysical_member_is_reported_by_its_call(port):
    oc, _ = both_configs("bubble", 1, False)
    o = port.mesh(oc).solver(3, "f64")
    good, bad = members_of(o, 2)
    bad = bad.copy()
    bad[5, 0, 7] = -1.0   # negative density in element 5, node 7
    _, s = make(port, "bubble", (1, False), 3, path=capi.PATH_STAGE)
    s.set_state(good)
    s.step_stream(1e-3, bad, None)            # steps `good`
    out = np.empty_like(good)
    with pytest.raises(capi.NonPhysicalState) as ei:
        s.step_stream(1e-3, good, out)        # steps `bad`
    assert ei.value.element == 5 and ei.value.node == 7 and ei.value.stage == 0
