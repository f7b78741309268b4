"""Level 1 of the C ABI driven directly (-m gpu), the way INTEGRATION.md
section 2 describes a reference-side binding that keeps its own mesh,
partition and exchange plan: every partition is an esdg_b200_shard built from
flattened host arrays, the caller moves the traces between the shards'
send / receive buffers itself and orders the kernels of rhs_job
(solver.hpp:240-340). Three partitions on cuda:0; the results are compared
bitwise with the level-2 solver on the undivided mesh."""
import ctypes as C

import numpy as np
import pytest
import torch

from oracle import pyoracle as po
from paper_2605_16684_b200 import capi, halo

pytestmark = pytest.mark.gpu

ORDER, WORLD = 3, 3
PARTS = (1, 2)   # ESDG_B200_PART_INTERIOR, _BOUNDARY


def face_trace(field, face, nq):
    """extract_phi_trace (kernels.hpp:340-345): FaceIndexer order fn = s + nq t,
    tangential axes (d+1)%3, (d+2)%3 (mesh.hpp:100-118)."""
    d, side = face >> 1, face & 1
    pitch = (1, nq, nq * nq)
    s, t = np.meshgrid(np.arange(nq), np.arange(nq), indexing="ij")
    n = side * (nq - 1) * pitch[d] + s * pitch[(d + 1) % 3] + t * pitch[(d + 2) % 3]
    out = np.empty(nq * nq, field.dtype)
    out[(s + nq * t).ravel()] = field[n.ravel()]
    return out


class Shard:
    def __init__(self, mesh, rank, phi, gas):
        lib = capi.lib()
        nq = ORDER + 1
        self.h_info = h = capi.rank_halo(mesh, WORLD, rank)
        self.begin, self.end = h["begin"], h["end"]
        nloc, nghost = self.end - self.begin, len(h["send_elem"])
        nodes, w, D = capi.reference_element(ORDER)
        cfg = mesh.cfg
        cells = np.array(cfg.base[:], np.int64) << cfg.refinement
        delta = (np.array(cfg.hi[:]) - np.array(cfg.lo[:])) / cells
        nbr_global = mesh.neighbors
        ghost_phi = np.empty((max(nghost, 1), nq * nq))
        for g in range(nghost):     # build_ghost_phi, solver.hpp:178-191
            face = int(h["send_face"][g])
            remote = int(nbr_global[self.begin + int(h["send_elem"][g]), face])
            ghost_phi[g] = face_trace(phi[remote], face ^ 1, nq)
        self.keep = dict(D=np.ascontiguousarray(D.ravel()), w=np.ascontiguousarray(w),
                         nbr=np.ascontiguousarray(h["nbr_local"], np.int32),
                         phi=np.ascontiguousarray(phi[self.begin:self.end]),
                         gphi=np.ascontiguousarray(ghost_phi),
                         se=np.ascontiguousarray(h["send_elem"], np.int32),
                         sf=np.ascontiguousarray(h["send_face"], np.int32))
        k = self.keep
        d = capi.ShardDesc()
        d.precision, d.nq, d.device, d.dissipation = 8, nq, 0, 1
        d.n_elements, d.elem_offset = nloc, self.begin
        d.diff = k["D"].ctypes.data_as(C.POINTER(C.c_double))
        d.weights = k["w"].ctypes.data_as(C.POINTER(C.c_double))
        d.metric[:] = list(2.0 / delta)
        d.gamma, d.gas_R = gas.gamma, gas.R
        d.coriolis_mode, d.n_ylevels = 0, 0
        d.nbr = k["nbr"].ctypes.data_as(C.POINTER(C.c_int32))
        d.phi = k["phi"].ctypes.data_as(C.c_void_p)
        d.n_ghost = d.n_send = nghost
        d.ghost_phi = k["gphi"].ctypes.data_as(C.c_void_p)
        d.send_elem = k["se"].ctypes.data_as(C.POINTER(C.c_int32))
        d.send_face = k["sf"].ctypes.data_as(C.POINTER(C.c_int32))
        self.s = C.c_void_p()
        capi.check(lib.esdg_b200_shard_create(C.byref(d), C.byref(self.s)))
        n = nghost * 5 * nq * nq
        self.send = halo.device_tensor(lib.esdg_b200_shard_send_ptr(self.s), n, torch.float64, 0)
        self.recv = halo.device_tensor(lib.esdg_b200_shard_recv_ptr(self.s), n, torch.float64, 0)
        self.trace = 5 * nq * nq
        self.shape = (nloc, 5, nq ** 3)

    def close(self):
        self.send = self.recv = None
        capi.lib().esdg_b200_shard_destroy(self.s)

    def upload(self, reg, a):
        a = np.ascontiguousarray(a[self.begin:self.end])
        capi.check(capi.lib().esdg_b200_shard_upload(self.s, reg, a.ctypes.data_as(C.c_void_p), 0, len(a)))

    def download(self, reg):
        out = np.empty(self.shape)
        capi.check(capi.lib().esdg_b200_shard_download(self.s, reg, out.ctypes.data_as(C.c_void_p), 0,
                                                       self.shape[0]))
        return out


def exchange(shards):
    """Transport::send / wait (exchange.hpp:32-57): pack on every shard, then
    every peer block moves from the sender's send buffer to the receiver's
    receive buffer (both ends enumerate the faces of a block identically)."""
    lib = capi.lib()
    for sh in shards:
        capi.check(lib.esdg_b200_shard_pack(sh.s, capi.REG_Q, None))
    torch.cuda.synchronize()
    for r, sh in enumerate(shards):
        for peer, off, cnt in sh.h_info["peers"]:
            poff = next(o for p, o, _ in shards[peer].h_info["peers"] if p == r)
            sh.recv[off * sh.trace:(off + cnt) * sh.trace].copy_(
                shards[peer].send[poff * sh.trace:(poff + cnt) * sh.trace])
    torch.cuda.synchronize()


@pytest.fixture()
def setup():
    mesh = capi.Mesh(capi.bubble_mesh_config(2, True))      # 64 elements, periodic in z too
    ref = capi.GpuSolver(mesh, ORDER, "f64")
    phi = ref.get_phi()
    q = po.Oracle("port").mesh(po.bubble_mesh_config(2, True)).solver(ORDER, "f64").init_case(
        po.CASE_ENTROPY_TEST, 77).copy()
    shards = [Shard(mesh, r, phi, ref.gas) for r in range(WORLD)]
    yield mesh, ref, q, shards
    torch.cuda.synchronize()
    for sh in shards:
        sh.close()


def gather(shards, reg):
    torch.cuda.synchronize()
    return np.concatenate([sh.download(reg) for sh in shards])


def test_shard_abi_rhs_orders(setup):
    """volume + surface, the one-pass kernel, and the one-pass kernel split
    into interior and boundary element groups all reproduce the solver's RHS."""
    lib = capi.lib()
    mesh, ref, q, shards = setup
    ref.set_path(capi.PATH_SPLIT)
    ref.set_state(q)
    ref.rhs(0.0, 1.0)
    want = ref.get_state(capi.REG_K)
    for sh in shards:
        sh.upload(capi.REG_Q, q)
    exchange(shards)
    for sh in shards:                                       # rhs_job's order, split path
        capi.check(lib.esdg_b200_shard_volume(sh.s, capi.REG_Q, capi.REG_K, 0.0, 1.0, 1, 0, None))
        capi.check(lib.esdg_b200_shard_surface(sh.s, capi.REG_Q, capi.REG_K, 1.0, 0, None))
    assert np.array_equal(gather(shards, capi.REG_K), want)
    ref.set_path(capi.PATH_FUSED)
    ref.rhs(0.0, 1.0)
    want = ref.get_state(capi.REG_K)
    for sh in shards:
        capi.check(lib.esdg_b200_shard_rhs_fused(sh.s, capi.REG_Q, capi.REG_K, 0.0, 1.0, 0, None))
    assert np.array_equal(gather(shards, capi.REG_K), want)
    counts = []
    for sh in shards:
        n = [C.c_int64(), C.c_int64(), C.c_int64()]
        for part in range(3):
            capi.check(lib.esdg_b200_shard_part_elements(sh.s, part, C.byref(n[part])))
        assert n[0].value == sh.shape[0] == n[1].value + n[2].value and n[2].value > 0
        counts.append(n[1].value)
        capi.check(lib.esdg_b200_shard_upload(sh.s, capi.REG_K, np.full(sh.shape, np.nan).ctypes.data_as(C.c_void_p),
                                              0, sh.shape[0]))
        for part in PARTS:
            capi.check(lib.esdg_b200_shard_rhs_fused_part(sh.s, capi.REG_Q, capi.REG_K, 0.0, 1.0, 0, part, None))
    assert np.array_equal(gather(shards, capi.REG_K), want)
    bad = C.c_int64()
    assert lib.esdg_b200_shard_part_elements(shards[0].s, 3, C.byref(bad)) == capi.BADARG
    assert lib.esdg_b200_shard_rhs_fused_part(shards[0].s, capi.REG_Q, capi.REG_K, 0.0, 1.0, 0, 7, None) == capi.BADARG


def test_shard_abi_lsrk_steps(setup):
    """Two LSRK steps with one kernel per stage and partition, interior groups
    before the traces are needed and boundary groups after (lsrk_step,
    time_integration.hpp:43-49), against esdg_b200_solver_step."""
    lib = capi.lib()
    mesh, ref, q, shards = setup
    a, b, _ = capi.lsrk_coefficients()
    dt = 1e-3
    ref.set_path(capi.PATH_STAGE)
    ref.set_state(q)
    for sh in shards:
        sh.upload(capi.REG_Q, q)
    for _ in range(2):
        ref.step(dt)
        for s in range(5):
            for sh in shards:
                capi.check(lib.esdg_b200_shard_pack(sh.s, capi.REG_Q, None))
            for sh in shards:       # no ghost face in these groups: they may run before the traces move
                capi.check(lib.esdg_b200_shard_stage_fused_part(sh.s, a[s], dt, b[s], s, 1, None))
            exchange(shards)        # (packs again: harmless, q is unchanged until the buffers swap)
            for sh in shards:
                capi.check(lib.esdg_b200_shard_stage_fused_part(sh.s, a[s], dt, b[s], s, 2, None))
        err = capi.Error()
        for sh in shards:
            assert lib.esdg_b200_shard_check(sh.s, None, C.byref(err)) == capi.OK
    assert np.array_equal(gather(shards, capi.REG_Q), ref.get_state())
    assert np.array_equal(gather(shards, capi.REG_K), ref.get_state(capi.REG_K))


def test_shard_abi_irregular_launch_sequences(setup):
    """The lift terms shared between elements carry the parity of the RHS
    evaluation they belong to (tagged lift terms, esdg_kernels.cuh); the shard
    keeps the parity consistent across the launches of one evaluation. Launch
    sequences that break the pattern -- an interior launch never followed by
    its boundary launch, an interior launch repeated, evaluations of
    different shapes back to back -- must still give the one-launch result,
    bitwise, afterwards. (A boundary launch always follows its interior
    launch: its groups pull terms the interior groups push.)"""
    lib = capi.lib()
    mesh, ref, q, shards = setup
    ref.set_path(capi.PATH_FUSED)
    ref.set_state(q)
    ref.rhs(0.0, 1.0)
    want = ref.get_state(capi.REG_K)
    for sh in shards:
        sh.upload(capi.REG_Q, q)
    exchange(shards)

    def full():
        for sh in shards:
            capi.check(lib.esdg_b200_shard_rhs_fused(sh.s, capi.REG_Q, capi.REG_K, 0.0, 1.0, 0, None))

    def part(p):
        for sh in shards:
            capi.check(lib.esdg_b200_shard_rhs_fused_part(sh.s, capi.REG_Q, capi.REG_K, 0.0, 1.0, 0, p, None))

    def poison():
        for sh in shards:
            capi.check(lib.esdg_b200_shard_upload(sh.s, capi.REG_K, np.full(sh.shape, np.nan).ctypes.data_as(C.c_void_p),
                                                  0, sh.shape[0]))

    def parts():
        part(1)
        part(2)

    # (what came before, the complete evaluation whose result is checked)
    sequences = [
        ([full, full], full),                          # alternating parities
        ([], parts),
        ([lambda: part(1)], full),                     # abandoned evaluation, then a whole one
        ([lambda: part(1), lambda: part(1)], parts),
        ([full, parts, full], parts),
        ([parts, parts, lambda: part(1)], parts),
    ]
    err = capi.Error()
    for before, final in sequences:
        for launch in before:
            launch()
        poison()
        final()
        assert np.array_equal(gather(shards, capi.REG_K), want)
        for sh in shards:
            assert lib.esdg_b200_shard_check(sh.s, None, C.byref(err)) == capi.OK
