"""ctypes bindings for the checker libraries under oracle/.

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs. The product package never
imports this module.

Two backends expose the same Python interface:
  * ``Oracle("port")``      -> oracle/liboracle.so       (the C restatement)
  * ``Oracle("reference")`` -> oracle/_ref/libesdg_ref.so (the unmodified
    reference compiled from /root/reference, see oracle/Makefile)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

CASE_BUBBLE_SHARP, CASE_BUBBLE_SMOOTH, CASE_HYDROSTATIC, CASE_ENTROPY_TEST, CASE_CONSTANT = range(5)


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
                ("slot", C.c_int32), ("my_inbox", C.c_int32),
                ("peer_inbox", C.c_int32)]


class Gas(C.Structure):
    _fields_ = [("gamma", C.c_double), ("R", C.c_double), ("p0", C.c_double),
                ("gravity", C.c_double)]


class Settings(C.Structure):
    _fields_ = [("dissipation", C.c_int32), ("coriolis_mode", C.c_int32),
                ("f0", C.c_double), ("beta", C.c_double), ("y0", C.c_double)]


class Error(C.Structure):
    _fields_ = [("set", C.c_int32), ("rho", C.c_double), ("pressure", C.c_double),
                ("element", C.c_int32), ("node", C.c_int32), ("stage", C.c_int32)]


def mesh_config(base=(1, 1, 1), refinement=0, lo=(0., 0., 0.), hi=(1., 1., 1.),
                bc=(0, 0, 0)) -> MeshConfig:
    c = MeshConfig()
    c.base[:] = base
    c.refinement = refinement
    c.lo[:] = lo
    c.hi[:] = hi
    c.bc[:] = bc
    return c


def bubble_mesh_config(refinement, periodic_z=False, base=(1, 1, 1)) -> MeshConfig:
    """tests/test_helpers.hpp:10-21 of the reference."""
    return mesh_config(base, refinement, (-1000., -1000., 0.), (1000., 1000., 2000.),
                       (0, 0, 0 if periodic_z else 1))


def unit_mesh_config(refinement) -> MeshConfig:
    """tests/test_helpers.hpp:23-29 of the reference."""
    return mesh_config((1, 1, 1), refinement)


def default_gas(gravity=9.81) -> Gas:
    return Gas(1.4, 287.0, 1e5, gravity)


def make_settings(dissipation=True, coriolis_mode=0, f0=0.0, beta=0.0, y0=0.0) -> Settings:
    return Settings(int(dissipation), coriolis_mode, f0, beta, y0)


def build(force=False):
    """Compile liboracle.so (and _ref when the reference tree is present)."""
    lib = os.path.join(HERE, "liboracle.so")
    if force or not os.path.exists(lib) or \
            os.path.getmtime(lib) < max(os.path.getmtime(os.path.join(HERE, f))
                                        for f in ("esdg_oracle.c", "esdg_oracle_impl.inc", "esdg_oracle.h")):
        subprocess.run(["make", "-C", HERE, "-s", os.path.join(HERE, "liboracle.so")], check=True)
    if os.path.isdir("/root/reference/proj/core"):
        subprocess.run(["make", "-C", HERE, "-s", "ref"], check=True)


def reference_available(fast=False) -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libesdg_ref_v3.so" if fast else "libesdg_ref.so"))


class _Owned(np.ndarray):
    """ndarray view of memory owned by a C handle; keeps the Python owner of
    that handle alive for as long as the view (or any view of it) lives."""

    def __array_finalize__(self, obj):
        self._owner = getattr(obj, "_owner", None)


def _owned(ptr, shape, owner):
    a = np.ctypeslib.as_array(ptr, shape=shape).view(_Owned)
    a._owner = owner
    return a


def _np_dtype(precision):
    return np.float64 if precision == "f64" else np.float32


def _c_real(precision):
    return C.c_double if precision == "f64" else C.c_float


class Oracle:
    """One loaded checker library ("port" or "reference")."""

    def __init__(self, kind="port", fast=False):
        self.kind = kind
        if kind == "port":
            build()
            path, self.p = os.path.join(HERE, "liboracle.so"), "orc_"
        elif kind == "reference":
            path = os.path.join(HERE, "_ref", "libesdg_ref_v3.so" if fast else "libesdg_ref.so")
            self.p = "ref_"
            if not os.path.exists(path):
                raise FileNotFoundError(path)
        else:
            raise ValueError(kind)
        self.lib = C.CDLL(path)
        self._declare()

    def f(self, name):
        return getattr(self.lib, self.p + name)

    def _declare(self):
        L, P = self.lib, self.p
        vp = C.c_void_p
        def sig(name, res, args):
            fn = getattr(L, P + name)
            fn.restype, fn.argtypes = res, args
        sig("mesh_create", vp, [C.POINTER(MeshConfig)])
        sig("mesh_destroy", None, [vp])
        sig("mesh_num_elements", C.c_int64, [vp])
        sig("mesh_num_faces", C.c_int32, [vp])
        sig("mesh_lattice", C.POINTER(C.c_int32), [vp])
        sig("mesh_faces", C.POINTER(Face), [vp])
        sig("mesh_face_of", C.POINTER(C.c_int32), [vp])
        sig("mesh_jacobian", C.c_double, [vp])
        dp = C.POINTER(C.c_double)
        sig("reference_element", C.c_int, [C.c_int, dp, dp, dp])
        sig("schedule", C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_int16),
                                  C.POINTER(C.c_int16), C.POINTER(C.c_int32)])
        sig("partition", C.c_int, [C.c_int64, C.c_int, C.POINTER(C.c_int64)])
        sig("exchange_plan", C.c_int, [vp, C.c_int, C.POINTER(C.c_int32),
                                       C.POINTER(C.c_int32), C.POINTER(GhostFace),
                                       C.POINTER(C.c_int32)])
        sig("lsrk_coefficients", None, [dp, dp, dp])
        for suf, R in (("f64", C.c_double), ("f32", C.c_float)):
            rp = C.POINTER(R)
            create_args = [vp, C.c_int, C.POINTER(Gas), C.POINTER(Settings)]
            if self.kind == "reference":
                create_args.append(C.c_int)
            sig(f"solver_create_{suf}", vp, create_args)
            sig(f"solver_destroy_{suf}", None, [vp])
            sig(f"solver_n3_{suf}", C.c_int, [vp])
            sig(f"solver_state_{suf}", rp, [vp])
            sig(f"solver_phi_{suf}", rp, [vp])
            sig(f"solver_ops_{suf}", None, [vp, rp, rp, rp, rp, rp])
            sig(f"solver_set_settings_{suf}", None, [vp, C.POINTER(Settings)])
            sig(f"solver_init_case_{suf}", C.c_int, [vp, C.c_int, C.c_uint64, dp])
            sig(f"assemble_rhs_{suf}", C.c_int, [vp, rp, rp, R, R])
            sig(f"volume_rhs_{suf}", C.c_int, [vp, rp, rp])
            sig(f"step_{suf}", C.c_int, [vp, R])
            sig(f"compute_dt_{suf}", C.c_double, [vp, C.c_double])
            sig(f"last_error_{suf}", None, [vp, C.POINTER(Error)])
            sig(f"quadrature_total_{suf}", C.c_double, [vp, rp, C.c_int])
            sig(f"total_entropy_{suf}", C.c_double, [vp, rp])
            sig(f"entropy_production_{suf}", C.c_double, [vp, rp, rp])
            sig(f"log_mean_{suf}", R, [R, R, R, R])
            sig(f"node_vals_{suf}", C.c_int, [rp, R, R, rp])
            sig(f"ec_flux_{suf}", None, [rp, rp, C.c_int, R, rp])
            sig(f"matrix_dissipation_{suf}", None, [rp, rp, C.c_int, R, R, rp])
            if self.kind == "port":
                sig(f"solver_kreg_{suf}", rp, [vp])
                sig(f"assemble_rhs_rank_{suf}", C.c_int,
                    [vp, rp, rp, R, R, C.c_int64, C.c_int64, C.POINTER(C.c_int32), rp])
                sig(f"extract_trace_{suf}", None, [vp, rp, C.c_int64, C.c_int, C.c_int, rp])
                sig(f"axpy_{suf}", None, [vp, R])
                sig(f"flux_scale_{suf}", C.c_int, [vp, rp, dp])
                sig(f"flux_scale_rank_{suf}", C.c_int,
                    [vp, rp, C.c_int64, C.c_int64, C.POINTER(C.c_int32), rp, dp])
            else:
                sig(f"perf_{suf}", None, [vp, dp, C.POINTER(C.c_uint64), C.c_int])
        if self.kind == "port":
            sig("fnv1a64", C.c_uint64, [vp, C.c_uint64])
            sig("morton_key", C.c_uint64, [C.c_uint32, C.c_uint32, C.c_uint32])
        else:
            sig("hardware_threads", C.c_int, [])

    # ---- free functions ---------------------------------------------------
    def reference_element(self, order):
        nq = order + 1
        x, w, d = np.zeros(nq), np.zeros(nq), np.zeros(nq * nq)
        dp = C.POINTER(C.c_double)
        rc = self.f("reference_element")(order, x.ctypes.data_as(dp), w.ctypes.data_as(dp),
                                         d.ctypes.data_as(dp))
        if rc != 0:
            raise ValueError("bad order")
        return x, w, d.reshape(nq, nq)

    def schedule(self, nq, variant=1):
        idx = np.zeros(nq * nq, np.int16)
        hw = np.zeros(nq * nq, np.int16)
        off = np.zeros(nq + 1, np.int32)
        n = self.f("schedule")(nq, variant, idx.ctypes.data_as(C.POINTER(C.c_int16)),
                               hw.ctypes.data_as(C.POINTER(C.c_int16)),
                               off.ctypes.data_as(C.POINTER(C.c_int32)))
        if n < 0:
            raise ValueError("bad nq")
        return idx[:n].copy(), hw[:n].copy(), off

    def partition(self, ne, ranks):
        rb = np.zeros(ranks + 1, np.int64) if ranks >= 0 else np.zeros(1, np.int64)
        rc = self.f("partition")(ne, ranks, rb.ctypes.data_as(C.POINTER(C.c_int64)))
        if rc != 0:
            raise ValueError("bad partition")
        return rb

    def lsrk(self):
        a, b, c = np.zeros(5), np.zeros(5), np.zeros(5)
        dp = C.POINTER(C.c_double)
        self.f("lsrk_coefficients")(a.ctypes.data_as(dp), b.ctypes.data_as(dp), c.ctypes.data_as(dp))
        return a, b, c

    def mesh(self, cfg: MeshConfig) -> "Mesh":
        return Mesh(self, cfg)


def fnv1a64(arr: np.ndarray) -> int:
    """FNV-1a-64 over the raw bytes (BASELINE.md section 4 fingerprints)."""
    h = 0xcbf29ce484222325
    data = np.ascontiguousarray(arr).view(np.uint8).ravel()
    # vectorised is impossible (sequential dependency); go through the C port
    o = _default_port()
    return int(o.f("fnv1a64")(data.ctypes.data_as(C.c_void_p), data.size))


_PORT = None


def _default_port() -> Oracle:
    global _PORT
    if _PORT is None:
        _PORT = Oracle("port")
    return _PORT


class Mesh:
    def __init__(self, oracle: Oracle, cfg: MeshConfig):
        self.o, self.cfg = oracle, cfg
        self.h = oracle.f("mesh_create")(C.byref(cfg))
        if not self.h:
            raise ValueError("invalid mesh config")
        self.ne = int(oracle.f("mesh_num_elements")(self.h))
        self.nfaces = int(oracle.f("mesh_num_faces")(self.h))

    def __del__(self):
        if getattr(self, "h", None):
            self.o.f("mesh_destroy")(self.h)
            self.h = None

    @property
    def lattice(self):
        p = self.o.f("mesh_lattice")(self.h)
        return np.ctypeslib.as_array(p, shape=(self.ne, 3)).copy()

    @property
    def face_of(self):
        p = self.o.f("mesh_face_of")(self.h)
        return np.ctypeslib.as_array(p, shape=(self.ne, 6)).copy()

    @property
    def faces(self):
        """(nfaces, 5) int array: minus, plus, dir, minus_side, reflecting."""
        p = self.o.f("mesh_faces")(self.h)
        out = np.zeros((self.nfaces, 5), np.int64)
        for i in range(self.nfaces):
            f = p[i]
            out[i] = (f.minus_elem, f.plus_elem, f.dir, f.minus_side, f.reflecting)
        return out

    @property
    def jacobian(self):
        return float(self.o.f("mesh_jacobian")(self.h))

    def exchange_plan(self, ranks):
        gc = np.zeros(ranks, np.int32)
        ic = np.zeros(ranks, np.int32)
        ip = C.POINTER(C.c_int32)
        n = self.o.f("exchange_plan")(self.h, ranks, gc.ctypes.data_as(ip), ic.ctypes.data_as(ip), None, None)
        if n < 0:
            raise ValueError("bad plan")
        ghosts = (GhostFace * int(gc.sum()))()
        interior = np.zeros(int(ic.sum()), np.int32)
        n = self.o.f("exchange_plan")(self.h, ranks, gc.ctypes.data_as(ip), ic.ctypes.data_as(ip),
                                      ghosts, interior.ctypes.data_as(ip))
        g = np.array([(x.face, x.peer, x.my_side, x.slot, x.my_inbox, x.peer_inbox) for x in ghosts],
                     np.int64).reshape(-1, 6)
        return dict(n_mailboxes=n, ghost_count=gc, interior_count=ic, ghosts=g, interior=interior)

    def solver(self, order, precision="f64", gas=None, settings=None, ranks=1) -> "Solver":
        return Solver(self, order, precision, gas or default_gas(), settings or make_settings(), ranks)


class NonPhysicalState(RuntimeError):
    def __init__(self, err: Error):
        super().__init__(f"non-physical state rho={err.rho} p={err.pressure} element={err.element} "
                         f"node={err.node} stage={err.stage}")
        self.rho, self.pressure = err.rho, err.pressure
        self.element, self.node, self.stage = err.element, err.node, err.stage


class Solver:
    def __init__(self, mesh: Mesh, order, precision, gas: Gas, settings: Settings, ranks=1):
        self.mesh, self.o, self.order, self.prec = mesh, mesh.o, order, precision
        self.dtype, self.R = _np_dtype(precision), _c_real(precision)
        self.gas, self.settings = gas, settings
        args = [mesh.h, order, C.byref(gas), C.byref(settings)]
        if self.o.kind == "reference":
            args.append(ranks)
        self.h = self._f("solver_create")(*args)
        if not self.h:
            raise ValueError("solver_create failed")
        self.nq = order + 1
        self.n3 = int(self._f("solver_n3")(self.h))
        self.ne = mesh.ne
        self.shape = (self.ne, 5, self.n3)

    def _f(self, name):
        return self.o.f(f"{name}_{self.prec}")

    def __del__(self):
        if getattr(self, "h", None):
            self._f("solver_destroy")(self.h)
            self.h = None

    def _ptr(self, a):
        assert a.dtype == self.dtype and a.flags["C_CONTIGUOUS"]
        return a.ctypes.data_as(C.POINTER(self.R))

    @property
    def state(self) -> np.ndarray:
        """Writable view of the internal q register, shape (ne, 5, n3)."""
        p = self._f("solver_state")(self.h)
        return _owned(p, self.shape, self)

    @property
    def kreg(self) -> np.ndarray:
        p = self._f("solver_kreg")(self.h)
        return _owned(p, self.shape, self)

    @property
    def phi(self) -> np.ndarray:
        p = self._f("solver_phi")(self.h)
        return _owned(p, (self.ne, self.n3), self)

    def ops(self):
        nq = self.nq
        d, w = np.zeros(nq * nq, self.dtype), np.zeros(nq, self.dtype)
        metric, fc, jac = np.zeros(3, self.dtype), np.zeros(3, self.dtype), np.zeros(1, self.dtype)
        self._f("solver_ops")(self.h, self._ptr(d), self._ptr(w), self._ptr(metric), self._ptr(fc),
                              self._ptr(jac))
        return dict(d=d.reshape(nq, nq), w=w, metric=metric, face_coef=fc, jacobian=jac[0])

    def set_settings(self, settings: Settings):
        self.settings = settings
        self._f("solver_set_settings")(self.h, C.byref(settings))

    def init_case(self, case_id, iparam=0, dparam=None):
        d = np.ascontiguousarray(dparam if dparam is not None else np.zeros(5), np.float64)
        rc = self._f("solver_init_case")(self.h, case_id, iparam, d.ctypes.data_as(C.POINTER(C.c_double)))
        if rc != 0:
            raise ValueError("init_case failed")
        return self.state

    def _raise(self):
        e = Error()
        self._f("last_error")(self.h, C.byref(e))
        raise NonPhysicalState(e)

    def assemble_rhs(self, q, out=None, a_old=0.0, a_new=1.0):
        if out is None:
            out = np.zeros(self.shape, self.dtype)
        if self._f("assemble_rhs")(self.h, self._ptr(q), self._ptr(out), a_old, a_new):
            self._raise()
        return out

    def volume_rhs(self, q, out=None):
        if out is None:
            out = np.zeros(self.shape, self.dtype)
        if self._f("volume_rhs")(self.h, self._ptr(q), self._ptr(out)):
            self._raise()
        return out

    def assemble_rhs_rank(self, q, out, a_old, a_new, eb, ee, ghost_slot_of_face, ghost_traces):
        gs = np.ascontiguousarray(ghost_slot_of_face, np.int32)
        gt = np.ascontiguousarray(ghost_traces, self.dtype)
        if gt.size == 0:
            gt = np.zeros(1, self.dtype)
        if self._f("assemble_rhs_rank")(self.h, self._ptr(q), self._ptr(out), a_old, a_new, eb, ee,
                                        gs.ctypes.data_as(C.POINTER(C.c_int32)), self._ptr(gt)):
            self._raise()
        return out

    def extract_trace(self, q, elem, d, side):
        out = np.zeros((5, self.nq * self.nq), self.dtype)
        self._f("extract_trace")(self.h, self._ptr(q), elem, d, side, self._ptr(out))
        return out

    def axpy(self, b):
        self._f("axpy")(self.h, b)

    def step(self, dt):
        if self._f("step")(self.h, dt):
            self._raise()

    def compute_dt(self, courant=0.5):
        return float(self._f("compute_dt")(self.h, courant))

    def quadrature_total(self, q, var):
        return float(self._f("quadrature_total")(self.h, self._ptr(q), var))

    def total_entropy(self, q):
        return float(self._f("total_entropy")(self.h, self._ptr(q)))

    def entropy_production(self, q, rhs):
        return float(self._f("entropy_production")(self.h, self._ptr(q), self._ptr(rhs)))

    def flux_scale(self, q):
        s = np.zeros(5)
        if self._f("flux_scale")(self.h, self._ptr(q), s.ctypes.data_as(C.POINTER(C.c_double))):
            self._raise()
        return s

    def flux_scale_rank(self, q, eb, ee, ghost_slot_of_face, ghost_traces):
        gs = np.ascontiguousarray(ghost_slot_of_face, np.int32)
        gt = np.ascontiguousarray(ghost_traces, self.dtype)
        s = np.zeros(5)
        if self._f("flux_scale_rank")(self.h, self._ptr(q), eb, ee,
                                      gs.ctypes.data_as(C.POINTER(C.c_int32)), self._ptr(gt),
                                      s.ctypes.data_as(C.POINTER(C.c_double))):
            self._raise()
        return s

    def perf(self, reset=False):
        p = np.zeros(5)
        c = np.zeros(7, np.uint64)
        self._f("perf")(self.h, p.ctypes.data_as(C.POINTER(C.c_double)),
                        c.ctypes.data_as(C.POINTER(C.c_uint64)), int(reset))
        return dict(wall=p[0], volume=p[1], surface=p[2], update=p[3], steps=int(p[4]),
                    vol_flux=int(c[0]), vol_log=int(c[1]), vol_div=int(c[2]),
                    surf_flux=int(c[3]), surf_log=int(c[4]), surf_div=int(c[5]), rhs_calls=int(c[6]))

    # ---- pointwise ----------------------------------------------------------
    def log_mean(self, am, ap, lam, lap):
        return float(self._f("log_mean")(am, ap, lam, lap))

    def node_vals(self, q5, phi, gamma=1.4):
        q5 = np.ascontiguousarray(q5, self.dtype)
        out = np.zeros(8, self.dtype)
        rc = self._f("node_vals")(self._ptr(q5), phi, gamma, self._ptr(out))
        return rc, out

    def ec_flux(self, m8, p8, d, gamma=1.4):
        m8, p8 = np.ascontiguousarray(m8, self.dtype), np.ascontiguousarray(p8, self.dtype)
        out = np.zeros(7, self.dtype)
        self._f("ec_flux")(self._ptr(m8), self._ptr(p8), d, gamma, self._ptr(out))
        return out

    def matrix_dissipation(self, m8, p8, d, gamma=1.4, Rgas=287.0):
        m8, p8 = np.ascontiguousarray(m8, self.dtype), np.ascontiguousarray(p8, self.dtype)
        out = np.zeros(5, self.dtype)
        self._f("matrix_dissipation")(self._ptr(m8), self._ptr(p8), d, gamma, Rgas, self._ptr(out))
        return out
