"""ctypes binding of libesdg_b200.so (include/esdg_b200.h).

Python is plumbing here: tests and bench.py drive the C ABI through this
module; the product is the shared library (CUDA kernels + C++ host mirror of
the reference's Solver interface). There is no CPU fallback: compute entry
points need a B200 and fail loudly otherwise.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
# (development: ESDG_B200_LIB points tools/ab_probe.sh at another build of the same library)
LIB_PATH = os.environ.get("ESDG_B200_LIB") or os.path.join(CSRC, "libesdg_b200.so")

OK, NONPHYSICAL, CUDA, BADARG = 0, 1, 2, 3
REG_Q, REG_K = 0, 1
PATH_SPLIT, PATH_FUSED, PATH_STAGE = 0, 1, 2
REDUCE_ON_DEVICE, REDUCE_ON_HOST = 0, 1
(CASE_BUBBLE_SHARP, CASE_BUBBLE_SMOOTH, CASE_HYDROSTATIC, CASE_ENTROPY_TEST,
 CASE_CONSTANT, CASE_BAROCLINIC, CASE_BAROCLINIC_JET) = range(7)


class MeshConfig(C.Structure):
    _fields_ = [("base", C.c_int32 * 3), ("refinement", C.c_int32),
                ("lo", C.c_double * 3), ("hi", C.c_double * 3),
                ("bc", C.c_int32 * 3)]


class Face(C.Structure):
    _fields_ = [("minus_elem", C.c_int32), ("plus_elem", C.c_int32),
                ("dir", C.c_uint8), ("minus_side", C.c_uint8),
                ("reflecting", C.c_uint8), ("pad_", C.c_uint8)]


class GhostFace(C.Structure):
    _fields_ = [("face", C.c_int32), ("peer", C.c_int32), ("my_side", C.c_int32),
                ("slot", C.c_int32), ("my_inbox", C.c_int32), ("peer_inbox", C.c_int32)]


class Gas(C.Structure):
    _fields_ = [("gamma", C.c_double), ("R", C.c_double), ("p0", C.c_double),
                ("gravity", C.c_double)]


class Settings(C.Structure):
    _fields_ = [("dissipation", C.c_int32), ("coriolis_mode", C.c_int32),
                ("f0", C.c_double), ("beta", C.c_double), ("y0", C.c_double)]


class Error(C.Structure):
    _fields_ = [("set", C.c_int32), ("rho", C.c_double), ("pressure", C.c_double),
                ("element", C.c_int64), ("node", C.c_int32), ("stage", C.c_int32)]


class ShardDesc(C.Structure):
    _fields_ = [("precision", C.c_int32), ("nq", C.c_int32), ("device", C.c_int32),
                ("dissipation", C.c_int32), ("n_elements", C.c_int64),
                ("elem_offset", C.c_int64), ("diff", C.POINTER(C.c_double)),
                ("weights", C.POINTER(C.c_double)), ("metric", C.c_double * 3),
                ("gamma", C.c_double), ("gas_R", C.c_double),
                ("coriolis_mode", C.c_int32), ("n_ylevels", C.c_int32),
                ("elem_ylevel", C.POINTER(C.c_int32)), ("coriolis_f", C.c_void_p),
                ("nbr", C.POINTER(C.c_int32)), ("phi", C.c_void_p),
                ("n_ghost", C.c_int32), ("ghost_phi", C.c_void_p),
                ("n_send", C.c_int32), ("send_elem", C.POINTER(C.c_int32)),
                ("send_face", C.POINTER(C.c_int32))]


EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p)

# every symbol include/esdg_b200.h declares: name -> (restype, argtypes)
_vp, _i, _i64, _d = C.c_void_p, C.c_int, C.c_int64, C.c_double
_dp, _ip, _i64p = C.POINTER(C.c_double), C.POINTER(C.c_int32), C.POINTER(C.c_int64)
SIGNATURES = {
    "esdg_b200_abi_version": (_i, []),
    "esdg_b200_last_message": (C.c_char_p, []),
    "esdg_b200_device_count": (_i, []),
    "esdg_b200_shard_create": (_i, [C.POINTER(ShardDesc), C.POINTER(_vp)]),
    "esdg_b200_shard_destroy": (None, [_vp]),
    "esdg_b200_shard_upload": (_i, [_vp, _i, _vp, _i64, _i64]),
    "esdg_b200_shard_download": (_i, [_vp, _i, _vp, _i64, _i64]),
    "esdg_b200_shard_upload_async": (_i, [_vp, _i, _vp, _i64, _i64, _vp]),
    "esdg_b200_shard_download_async": (_i, [_vp, _i, _vp, _i64, _i64, _vp]),
    "esdg_b200_shard_register_ptr": (_vp, [_vp, _i]),
    "esdg_b200_shard_send_ptr": (_vp, [_vp]),
    "esdg_b200_shard_recv_ptr": (_vp, [_vp]),
    "esdg_b200_shard_stream": (_vp, [_vp]),
    "esdg_b200_shard_pack": (_i, [_vp, _i, _vp]),
    "esdg_b200_shard_volume": (_i, [_vp, _i, _i, _d, _d, _i, _i, _vp]),
    "esdg_b200_shard_surface": (_i, [_vp, _i, _i, _d, _i, _vp]),
    "esdg_b200_shard_rhs_fused": (_i, [_vp, _i, _i, _d, _d, _i, _vp]),
    "esdg_b200_shard_stage_fused": (_i, [_vp, _d, _d, _d, _i, _vp]),
    "esdg_b200_shard_rhs_fused_part": (_i, [_vp, _i, _i, _d, _d, _i, _i, _vp]),
    "esdg_b200_shard_stage_fused_part": (_i, [_vp, _d, _d, _d, _i, _i, _vp]),
    "esdg_b200_shard_part_elements": (_i, [_vp, _i, C.POINTER(C.c_int64)]),
    "esdg_b200_shard_axpy": (_i, [_vp, _d, _vp]),
    "esdg_b200_shard_check": (_i, [_vp, _vp, C.POINTER(Error)]),
    "esdg_b200_shard_reduce": (_i, [_vp, _i, _i, _i, _dp, _dp, _d, _dp, C.POINTER(C.c_int32)]),
    "esdg_b200_shard_launch_count": (_i64, [_vp]),
    "esdg_b200_mesh_create": (_i, [C.POINTER(MeshConfig), C.POINTER(_vp)]),
    "esdg_b200_mesh_destroy": (None, [_vp]),
    "esdg_b200_mesh_num_elements": (_i64, [_vp]),
    "esdg_b200_mesh_num_faces": (_i64, [_vp]),
    "esdg_b200_mesh_lattice": (_ip, [_vp]),
    "esdg_b200_mesh_faces": (C.POINTER(Face), [_vp]),
    "esdg_b200_mesh_face_of": (_ip, [_vp]),
    "esdg_b200_mesh_neighbors": (_ip, [_vp]),
    "esdg_b200_reference_element": (_i, [_i, _dp, _dp, _dp]),
    "esdg_b200_partition": (_i, [_i64, _i, _i64p]),
    "esdg_b200_exchange_plan": (_i, [_vp, _i, _ip, _ip, C.POINTER(GhostFace), _ip]),
    "esdg_b200_rank_halo": (_i, [_vp, _i, _i, _ip, _i64p, _ip, _i64p, _i64p, _ip, _ip, _ip]),
    "esdg_b200_lsrk_coefficients": (None, [_dp, _dp, _dp]),
    "esdg_b200_solver_create": (_i, [_vp, _i, C.POINTER(Gas), C.POINTER(Settings), _i, _i,
                                     _ip, _i, C.POINTER(_vp)]),
    "esdg_b200_solver_create_distributed": (_i, [_vp, _i, C.POINTER(Gas), C.POINTER(Settings),
                                                 _i, _i, _i, _i, EXCHANGE_FN, _vp,
                                                 C.POINTER(_vp)]),
    "esdg_b200_nccl_unique_id": (_i, [_vp]),
    "esdg_b200_solver_create_nccl": (_i, [_vp, _i, C.POINTER(Gas), C.POINTER(Settings),
                                          _i, _i, _i, _i, _vp, C.POINTER(_vp)]),
    "esdg_b200_solver_nccl_version": (_i, [_vp]),
    "esdg_b200_solver_set_variant": (_i, [_vp, _i]),
    "esdg_b200_solver_record_events": (_i, [_vp, _i]),
    "esdg_b200_solver_rank_events": (_i, [_vp, _i, _i64p]),
    "esdg_b200_solver_halo_bytes": (_i64, [_vp]),
    "esdg_b200_solver_set_exchange_delay": (_i, [_vp, _i]),
    "esdg_b200_solver_destroy": (None, [_vp]),
    "esdg_b200_solver_set_path": (_i, [_vp, _i]),
    "esdg_b200_face_roles": (_i, [_ip, _i64, _i, _i, _vp]),
    "esdg_b200_nccl_selftest": (_i, [_i, _i, _i64, _i64p]),
    "esdg_b200_solver_set_overlap": (_i, [_vp, _i]),
    "esdg_b200_solver_set_face_sharing": (_i, [_vp, _i]),
    "esdg_b200_solver_overlap_elements": (_i, [_vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "esdg_b200_solver_set_settings": (_i, [_vp, C.POINTER(Settings)]),
    "esdg_b200_solver_local_begin": (_i64, [_vp]),
    "esdg_b200_solver_local_end": (_i64, [_vp]),
    "esdg_b200_solver_n3": (_i, [_vp]),
    "esdg_b200_solver_halo": (_i, [_vp, _ip, _i64p, _i64p, _i]),
    "esdg_b200_solver_stream": (_vp, [_vp]),
    "esdg_b200_solver_send_ptr": (_vp, [_vp]),
    "esdg_b200_solver_recv_ptr": (_vp, [_vp]),
    "esdg_b200_solver_n_ghost": (_i64, [_vp]),
    "esdg_b200_solver_init_case": (_i, [_vp, _i, C.c_uint64, _dp]),
    "esdg_b200_case_point": (_i, [_i, _vp, _vp, _vp, C.c_uint64, _dp, _d, _d, _d, _dp]),
    "esdg_b200_solver_set_state": (_i, [_vp, _i, _vp]),
    "esdg_b200_solver_get_state": (_i, [_vp, _i, _vp]),
    "esdg_b200_solver_swap_state": (_i, [_vp, _i, _vp, _vp]),
    "esdg_b200_solver_step_swap": (_i, [_vp, _d, _vp, _vp, _i]),
    "esdg_b200_solver_step_stream": (_i, [_vp, _d, _vp, _vp, _i]),
    "esdg_b200_solver_stream_collect": (_i, [_vp, _vp]),
    "esdg_b200_solver_get_phi": (_i, [_vp, _vp]),
    "esdg_b200_solver_assemble_rhs": (_i, [_vp, _vp, _vp, _d, _d]),
    "esdg_b200_solver_volume_rhs": (_i, [_vp, _vp, _vp]),
    "esdg_b200_solver_rhs": (_i, [_vp, _d, _d, _i]),
    "esdg_b200_solver_axpy": (_i, [_vp, _d]),
    "esdg_b200_solver_step": (_i, [_vp, _d, _i]),
    "esdg_b200_solver_sync": (_i, [_vp]),
    "esdg_b200_solver_compute_dt": (_i, [_vp, _d, _dp]),
    "esdg_b200_solver_last_error": (_i, [_vp, C.POINTER(Error)]),
    "esdg_b200_solver_quadrature_total": (_i, [_vp, _i, _i, _dp]),
    "esdg_b200_solver_total_entropy": (_i, [_vp, _dp]),
    "esdg_b200_solver_set_reduction": (_i, [_vp, _i]),
    "esdg_b200_solver_entropy_production": (_i, [_vp, _dp]),
    "esdg_b200_solver_enable_timing": (_i, [_vp, _i]),
    "esdg_b200_solver_timers": (_i, [_vp, _dp, _i64p, _i]),
    "esdg_b200_measure_fma_peak": (_i, [_i, _i, _dp]),
    "esdg_b200_measure_fma3_peak": (_i, [_i, _i, _dp]),
    "esdg_b200_selftest": (_i, [_i, _i, _dp]),
}


def build_library(force: bool = False) -> str:
    """Compiles csrc/ into libesdg_b200.so for sm_100a (nvcc, no GPU needed)."""
    if force:
        subprocess.run(["make", "-C", CSRC, "clean"], check=True, capture_output=True)
    subprocess.run(["make", "-C", CSRC, "-j", str(os.cpu_count() or 4)], check=True,
                   capture_output=True)
    return LIB_PATH


_LIB = None


def lib() -> C.CDLL:
    """The loaded library. Fails loudly when it has not been built."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: run __graft_entry__.build() (make -C {CSRC}). "
                "There is no CPU fallback for the ESDG right-hand side.")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        _LIB = L
    return _LIB


class EsdgError(RuntimeError):
    pass


class NonPhysicalState(EsdgError):
    def __init__(self, err: Error):
        super().__init__(f"non-physical state (rho={err.rho}, p={err.pressure}) at element="
                         f"{err.element} node={err.node} stage={err.stage}")
        self.rho, self.pressure = err.rho, err.pressure
        self.element, self.node, self.stage = err.element, err.node, err.stage


def check(rc: int, solver=None):
    if rc == OK:
        return
    if rc == NONPHYSICAL and solver is not None:
        e = Error()
        lib().esdg_b200_solver_last_error(solver, C.byref(e))
        raise NonPhysicalState(e)
    msg = lib().esdg_b200_last_message().decode()
    raise EsdgError(f"esdg_b200 status {rc}: {msg}")


def mesh_config(base=(1, 1, 1), refinement=0, lo=(0., 0., 0.), hi=(1., 1., 1.),
                bc=(0, 0, 0)) -> MeshConfig:
    c = MeshConfig()
    c.base[:] = base
    c.refinement = refinement
    c.lo[:] = lo
    c.hi[:] = hi
    c.bc[:] = bc
    return c


def bubble_mesh_config(refinement, periodic_z=False, base=(1, 1, 1), scale=(1, 1, 1)) -> MeshConfig:
    """bubble_mesh of the reference's tests/test_helpers.hpp:10-21; `scale`
    stretches the 2 km box with the base lattice (weak-scaling configs)."""
    return mesh_config(base, refinement,
                       (-1000. * scale[0], -1000. * scale[1], 0.),
                       (1000. * scale[0], 1000. * scale[1], 2000. * scale[2]),
                       (0, 0, 0 if periodic_z else 1))


def channel_mesh_config(refinement, base=(12, 2, 1)) -> MeshConfig:
    """case_defaults(BaroclinicChannel), core/src/config.cpp:84-95."""
    return mesh_config(base, refinement, (0., 0., 0.), (4e7, 6e6, 3e4), (0, 1, 1))


def case_point(case_id, cfg: MeshConfig, gas: "Gas", settings: "Settings | None", x, y, z,
               iparam=0, dparam=None):
    """The named initial state at one point (host only), as five doubles."""
    d = np.zeros(8)
    if dparam is not None:
        d[:len(dparam)] = dparam
    q = np.zeros(5)
    check(lib().esdg_b200_case_point(case_id, C.byref(cfg), C.byref(gas),
                                      C.byref(settings) if settings is not None else None,
                                      iparam, d.ctypes.data_as(_dp), x, y, z, q.ctypes.data_as(_dp)))
    return q


class Mesh:
    def __init__(self, cfg: MeshConfig):
        self.cfg = cfg
        h = C.c_void_p()
        check(lib().esdg_b200_mesh_create(C.byref(cfg), C.byref(h)))
        self.h = h
        self.ne = int(lib().esdg_b200_mesh_num_elements(h))

    def __del__(self):
        if getattr(self, "h", None):
            lib().esdg_b200_mesh_destroy(self.h)
            self.h = None

    @property
    def nfaces(self):
        return int(lib().esdg_b200_mesh_num_faces(self.h))

    @property
    def lattice(self):
        return np.ctypeslib.as_array(lib().esdg_b200_mesh_lattice(self.h), shape=(self.ne, 3)).copy()

    @property
    def neighbors(self):
        return np.ctypeslib.as_array(lib().esdg_b200_mesh_neighbors(self.h), shape=(self.ne, 6)).copy()

    @property
    def face_of(self):
        return np.ctypeslib.as_array(lib().esdg_b200_mesh_face_of(self.h), shape=(self.ne, 6)).copy()

    @property
    def faces(self):
        n = self.nfaces
        p = lib().esdg_b200_mesh_faces(self.h)
        out = np.zeros((n, 5), np.int64)
        for i in range(n):
            f = p[i]
            out[i] = (f.minus_elem, f.plus_elem, f.dir, f.minus_side, f.reflecting)
        return out

    def exchange_plan(self, ranks):
        gc, ic = np.zeros(ranks, np.int32), np.zeros(ranks, np.int32)
        n = lib().esdg_b200_exchange_plan(self.h, ranks, gc.ctypes.data_as(_ip), ic.ctypes.data_as(_ip),
                                          None, None)
        if n < 0:
            raise EsdgError("exchange_plan failed")
        ghosts = (GhostFace * max(1, int(gc.sum())))()
        interior = np.zeros(max(1, int(ic.sum())), np.int32)
        n = lib().esdg_b200_exchange_plan(self.h, ranks, gc.ctypes.data_as(_ip), ic.ctypes.data_as(_ip),
                                          ghosts, interior.ctypes.data_as(_ip))
        g = np.array([(x.face, x.peer, x.my_side, x.slot, x.my_inbox, x.peer_inbox)
                      for x in ghosts[:int(gc.sum())]], np.int64).reshape(-1, 6)
        return dict(n_mailboxes=n, ghost_count=gc, interior_count=ic, ghosts=g,
                    interior=interior[:int(ic.sum())].copy())


def rank_halo(mesh: Mesh, world_size: int, rank: int):
    """GPU-side halo lists of one partition (host only, no device needed)."""
    npeers, nghost = C.c_int32(), C.c_int64()
    check(lib().esdg_b200_rank_halo(mesh.h, world_size, rank, C.byref(npeers), C.byref(nghost),
                                    None, None, None, None, None, None))
    rb = partition(mesh.ne, world_size)
    nloc = int(rb[rank + 1] - rb[rank])
    peer = np.zeros(max(1, npeers.value), np.int32)
    off = np.zeros(max(1, npeers.value), np.int64)
    cnt = np.zeros(max(1, npeers.value), np.int64)
    se = np.zeros(max(1, nghost.value), np.int32)
    sf = np.zeros(max(1, nghost.value), np.int32)
    nbr = np.zeros((nloc, 6), np.int32)
    check(lib().esdg_b200_rank_halo(mesh.h, world_size, rank, C.byref(npeers), C.byref(nghost),
                                    peer.ctypes.data_as(_ip), off.ctypes.data_as(_i64p),
                                    cnt.ctypes.data_as(_i64p), se.ctypes.data_as(_ip),
                                    sf.ctypes.data_as(_ip), nbr.ctypes.data_as(_ip)))
    n, g = npeers.value, nghost.value
    return dict(begin=int(rb[rank]), end=int(rb[rank + 1]),
                peers=[(int(peer[i]), int(off[i]), int(cnt[i])) for i in range(n)],
                send_elem=se[:g].copy(), send_face=sf[:g].copy(), nbr_local=nbr)


def face_roles(nbr_local, elements_per_group, split=False):
    """Face roles of the one-pass kernels for a shard's neighbour codes (host
    only): bit f = face lf = 2f is pulled, bit 3 + d = face lf = 2d + 1 is
    pushed."""
    nbr = np.ascontiguousarray(nbr_local, np.int32)
    roles = np.zeros(max(1, nbr.shape[0]), np.uint8)
    check(lib().esdg_b200_face_roles(nbr.ctypes.data_as(_ip), nbr.shape[0], int(elements_per_group),
                                     1 if split else 0, roles.ctypes.data_as(_vp)))
    return roles[:nbr.shape[0]]


def reference_element(order):
    nq = order + 1
    x, w, d = np.zeros(nq), np.zeros(nq), np.zeros(nq * nq)
    check(lib().esdg_b200_reference_element(order, x.ctypes.data_as(_dp), w.ctypes.data_as(_dp),
                                            d.ctypes.data_as(_dp)))
    return x, w, d.reshape(nq, nq)


def partition(ne, ranks):
    rb = np.zeros(max(ranks, 0) + 1, np.int64)
    check(lib().esdg_b200_partition(ne, ranks, rb.ctypes.data_as(_i64p)))
    return rb


def lsrk_coefficients():
    a, b, c = np.zeros(5), np.zeros(5), np.zeros(5)
    lib().esdg_b200_lsrk_coefficients(a.ctypes.data_as(_dp), b.ctypes.data_as(_dp), c.ctypes.data_as(_dp))
    return a, b, c


class GpuSolver:
    """Handle on esdg_b200_solver: the GPU counterpart of esdg::Solver<Real>."""

    def __init__(self, mesh: Mesh, order, precision="f64", gas=None, settings=None, ranks=1,
                 devices=None, distributed=None, nccl=None):
        self.mesh, self.order = mesh, order
        self.prec = 8 if precision in ("f64", 8) else 4
        self.dtype = np.float64 if self.prec == 8 else np.float32
        self.gas = gas or Gas(1.4, 287.0, 1e5, 9.81)
        self.settings = settings or Settings(1, 0, 0.0, 0.0, 0.0)
        h = C.c_void_p()
        if nccl is not None:
            # one process per GPU, the exchange in the library (ncclSend/ncclRecv):
            # nccl = (world_size, rank, device, 128-byte unique id)
            world, rank, device, uid = nccl
            buf = (C.c_ubyte * 128).from_buffer_copy(bytes(uid))
            check(lib().esdg_b200_solver_create_nccl(
                mesh.h, order, C.byref(self.gas), C.byref(self.settings), self.prec, world, rank,
                device, buf, C.byref(h)))
        elif distributed is None:
            dev = np.ascontiguousarray(devices if devices is not None else [0], np.int32)
            check(lib().esdg_b200_solver_create(mesh.h, order, C.byref(self.gas), C.byref(self.settings),
                                                self.prec, ranks, dev.ctypes.data_as(_ip), dev.size,
                                                C.byref(h)))
        else:
            world, rank, device = distributed
            # late-bound trampoline: the exchange needs the solver's buffers,
            # which only exist after creation (see halo.make_exchange_callback)
            self.exchange_impl = None

            def _trampoline(user, phase, stream):
                if self.exchange_impl is None:
                    return 1
                return self.exchange_impl(user, phase, stream)

            self._cb = EXCHANGE_FN(_trampoline)
            check(lib().esdg_b200_solver_create_distributed(
                mesh.h, order, C.byref(self.gas), C.byref(self.settings), self.prec, world, rank,
                device, self._cb, None, C.byref(h)))
        self.h = h
        self.rank0 = 0 if (distributed is None and nccl is None) else (distributed or nccl)[1]
        self.n3 = int(lib().esdg_b200_solver_n3(h))
        self.nq = order + 1
        self.begin = int(lib().esdg_b200_solver_local_begin(h))
        self.end = int(lib().esdg_b200_solver_local_end(h))
        self.shape = (self.end - self.begin, 5, self.n3)

    def __del__(self):
        if getattr(self, "h", None):
            lib().esdg_b200_solver_destroy(self.h)
            self.h = None

    def _chk(self, rc):
        check(rc, self.h)

    def set_path(self, path):
        self._chk(lib().esdg_b200_solver_set_path(self.h, path))

    def set_variant(self, variant):
        """KernelVariant (kernels.hpp:27-34): 0 baseline .. 5 balanced."""
        self._chk(lib().esdg_b200_solver_set_variant(self.h, variant))

    def set_exchange_delay(self, microseconds):
        """Transport::send_hook analogue: hold every trace transfer back."""
        self._chk(lib().esdg_b200_solver_set_exchange_delay(self.h, int(microseconds)))

    def record_events(self, on=True):
        self._chk(lib().esdg_b200_solver_record_events(self.h, 1 if on else 0))

    def rank_events(self, rank=None):
        """RankEvents of the last recorded RHS of partition `rank` (default: the
        first local one), ns since that RHS was enqueued."""
        ns = np.zeros(5, np.int64)
        r = self.rank0 if rank is None else rank
        self._chk(lib().esdg_b200_solver_rank_events(self.h, r, ns.ctypes.data_as(_i64p)))
        return dict(zip(("sends_posted_ns", "volume_start_ns", "volume_end_ns", "wait_end_ns",
                         "last_arrival_ns"), (int(x) for x in ns)))

    @property
    def halo_bytes(self) -> int:
        return int(lib().esdg_b200_solver_halo_bytes(self.h))

    def set_overlap(self, on):
        self._chk(lib().esdg_b200_solver_set_overlap(self.h, 1 if on else 0))

    def set_face_sharing(self, on):
        self._chk(lib().esdg_b200_solver_set_face_sharing(self.h, 1 if on else 0))

    def overlap_elements(self):
        """(elements whose work hides the halo exchange, all local elements)"""
        a, b = C.c_int64(0), C.c_int64(0)
        self._chk(lib().esdg_b200_solver_overlap_elements(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def set_settings(self, settings: Settings):
        self._chk(lib().esdg_b200_solver_set_settings(self.h, C.byref(settings)))
        self.settings = settings

    def init_case(self, case_id, iparam=0, dparam=None):
        d = np.ascontiguousarray(dparam if dparam is not None else np.zeros(5), np.float64)
        d = np.concatenate([d, np.zeros(max(0, 5 - d.size))])
        self._chk(lib().esdg_b200_solver_init_case(self.h, case_id, iparam, d.ctypes.data_as(_dp)))

    def set_state(self, q, reg=REG_Q):
        q = np.ascontiguousarray(q, self.dtype)
        assert q.shape == self.shape
        self._chk(lib().esdg_b200_solver_set_state(self.h, reg, q.ctypes.data_as(_vp)))

    def get_state(self, reg=REG_Q):
        out = np.empty(self.shape, self.dtype)
        self._chk(lib().esdg_b200_solver_get_state(self.h, reg, out.ctypes.data_as(_vp)))
        return out

    def swap_state(self, q_in, q_out=None, reg=REG_Q):
        """Downloads the register into q_out and refills it from q_in in one
        full-duplex pass; q_out defaults to a new array, may be q_in itself."""
        q_in = np.ascontiguousarray(q_in, self.dtype)
        assert q_in.shape == self.shape
        if q_out is None:
            q_out = np.empty(self.shape, self.dtype)
        assert q_out.shape == self.shape and q_out.dtype == self.dtype and q_out.flags.c_contiguous
        self._chk(lib().esdg_b200_solver_swap_state(self.h, reg, q_in.ctypes.data_as(_vp),
                                                    q_out.ctypes.data_as(_vp)))
        return q_out

    def step_swap(self, dt, q_in, q_out=None, check_state=True):
        """One LSRK step, then the result to q_out and q_in in as the next
        state; finished parts of the last stage leave while it still runs."""
        q_in = np.ascontiguousarray(q_in, self.dtype)
        assert q_in.shape == self.shape
        if q_out is None:
            q_out = np.empty(self.shape, self.dtype)
        assert q_out.shape == self.shape and q_out.dtype == self.dtype and q_out.flags.c_contiguous
        self._chk(lib().esdg_b200_solver_step_swap(self.h, dt, q_in.ctypes.data_as(_vp),
                                                   q_out.ctypes.data_as(_vp), 1 if check_state else 0))
        return q_out

    def step_stream(self, dt, q_in_next=None, q_out_prev=None, check_state=True):
        """One LSRK step of the state on the device while q_in_next (the state
        of the next call, or None) is uploaded and the previous call's parked
        result is downloaded into q_out_prev (None when nothing is parked).
        The arrays are used in place: C-contiguous, the solver's dtype and shape
        (pinned memory for the transfers to overlap)."""
        for a in (q_in_next, q_out_prev):
            assert a is None or (a.shape == self.shape and a.dtype == self.dtype and a.flags.c_contiguous)
        self._chk(lib().esdg_b200_solver_step_stream(
            self.h, dt, None if q_in_next is None else q_in_next.ctypes.data_as(_vp),
            None if q_out_prev is None else q_out_prev.ctypes.data_as(_vp), 1 if check_state else 0))

    def stream_collect(self, q_out=None):
        """The parked result of the last step_stream call."""
        if q_out is None:
            q_out = np.empty(self.shape, self.dtype)
        assert q_out.shape == self.shape and q_out.dtype == self.dtype and q_out.flags.c_contiguous
        self._chk(lib().esdg_b200_solver_stream_collect(self.h, q_out.ctypes.data_as(_vp)))
        return q_out

    def get_phi(self):
        out = np.empty((self.shape[0], self.n3), self.dtype)
        self._chk(lib().esdg_b200_solver_get_phi(self.h, out.ctypes.data_as(_vp)))
        return out

    def assemble_rhs(self, q, out=None, a_old=0.0, a_new=1.0):
        q = np.ascontiguousarray(q, self.dtype)
        if out is None:
            out = np.zeros(self.shape, self.dtype)
        assert out.dtype == self.dtype and out.flags["C_CONTIGUOUS"]
        self._chk(lib().esdg_b200_solver_assemble_rhs(self.h, q.ctypes.data_as(_vp),
                                                      out.ctypes.data_as(_vp), a_old, a_new))
        return out

    def volume_rhs(self, q, out=None):
        q = np.ascontiguousarray(q, self.dtype)
        if out is None:
            out = np.zeros(self.shape, self.dtype)
        self._chk(lib().esdg_b200_solver_volume_rhs(self.h, q.ctypes.data_as(_vp), out.ctypes.data_as(_vp)))
        return out

    def rhs(self, a_old=0.0, a_new=1.0, stage=-1):
        self._chk(lib().esdg_b200_solver_rhs(self.h, a_old, a_new, stage))

    def axpy(self, b):
        self._chk(lib().esdg_b200_solver_axpy(self.h, b))

    def step(self, dt, check_state=True):
        self._chk(lib().esdg_b200_solver_step(self.h, dt, int(check_state)))

    def sync(self):
        self._chk(lib().esdg_b200_solver_sync(self.h))

    def compute_dt(self, courant=0.5):
        dt = C.c_double()
        self._chk(lib().esdg_b200_solver_compute_dt(self.h, courant, C.byref(dt)))
        return dt.value

    def set_reduction(self, mode):
        """REDUCE_ON_DEVICE (default) or REDUCE_ON_HOST (the reference's
        summation order, bitwise; moves the state to the host)."""
        self._chk(lib().esdg_b200_solver_set_reduction(self.h, mode))

    def quadrature_total(self, var, reg=REG_Q):
        v = C.c_double()
        self._chk(lib().esdg_b200_solver_quadrature_total(self.h, reg, var, C.byref(v)))
        return v.value

    def total_entropy(self):
        v = C.c_double()
        self._chk(lib().esdg_b200_solver_total_entropy(self.h, C.byref(v)))
        return v.value

    def entropy_production(self):
        v = C.c_double()
        self._chk(lib().esdg_b200_solver_entropy_production(self.h, C.byref(v)))
        return v.value

    def enable_timing(self, on=True):
        self._chk(lib().esdg_b200_solver_enable_timing(self.h, int(on)))

    def timers(self, reset=False):
        s = np.zeros(4)
        n = C.c_int64()
        self._chk(lib().esdg_b200_solver_timers(self.h, s.ctypes.data_as(_dp), C.byref(n), int(reset)))
        return dict(volume=s[0], surface=s[1], update=s[2], pack=s[3], launches=n.value)

    @property
    def stream(self) -> int:
        return int(lib().esdg_b200_solver_stream(self.h) or 0)

    @property
    def n_ghost(self) -> int:
        return int(lib().esdg_b200_solver_n_ghost(self.h))

    def halo_buffers(self):
        """(send_ptr, recv_ptr, bytes per trace) of a single-partition solver."""
        return (int(lib().esdg_b200_solver_send_ptr(self.h) or 0),
                int(lib().esdg_b200_solver_recv_ptr(self.h) or 0),
                self.prec * 5 * self.nq * self.nq)

    def halo(self):
        cap = 64
        peer, off, cnt = np.zeros(cap, np.int32), np.zeros(cap, np.int64), np.zeros(cap, np.int64)
        n = lib().esdg_b200_solver_halo(self.h, peer.ctypes.data_as(_ip), off.ctypes.data_as(_i64p),
                                        cnt.ctypes.data_as(_i64p), cap)
        return [(int(peer[i]), int(off[i]), int(cnt[i])) for i in range(n)]


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it, the host distributes it)."""
    buf = (C.c_ubyte * 128)()
    check(lib().esdg_b200_nccl_unique_id(buf))
    return bytes(buf)


def selftest(device=0, precision=8):
    out = np.zeros(5)
    check(lib().esdg_b200_selftest(device, precision, out.ctypes.data_as(_dp)))
    return dict(rcp_max_ulp=out[0], rcp_scaling_violations=int(out[1]), rcp_one_exact=bool(out[2]),
                samples=int(out[3]), log_vs_cuda_max_ulp=out[4])


def measure_fma_peak(device=0, precision=8, vector_operands=1) -> float:
    """FMA peak in TFLOP/s; vector_operands=3: three distinct vector registers
    per FMA (an sm_100 FP64 instruction of that shape takes 3 pipe cycles)."""
    v = C.c_double()
    fn = lib().esdg_b200_measure_fma3_peak if vector_operands >= 3 else lib().esdg_b200_measure_fma_peak
    check(fn(device, precision, C.byref(v)))
    return v.value
