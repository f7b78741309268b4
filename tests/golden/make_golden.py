"""Generates the golden vectors under tests/golden/ by RUNNING THE REFERENCE
(oracle/_ref/libesdg_ref.so, compiled from /root/reference by oracle/Makefile).
Run in the build container only; the fixtures are committed because
/root/reference does not exist on the GPU box.

    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import pyoracle as po  # noqa: E402

R = po.Oracle("reference")
arrays, kats = {}, {}

# --- BASELINE.json configs[0]: sharp bubble, bubble_mesh(3), N=4, FP64 -------
s = R.mesh(po.bubble_mesh_config(3)).solver(4, "f64")
q = s.init_case(po.CASE_BUBBLE_SHARP)
dt = s.compute_dt(0.5)
rhs0 = s.assemble_rhs(q.copy())
c1 = {"dt": dt, "rhs0_max_abs": [float(np.abs(rhs0[:, v]).max()) for v in range(5)],
      "rhs0_fnv": "%016x" % po.fnv1a64(rhs0), "steps": []}
for step in range(11):
    st = s.state.copy()
    rhs = s.assemble_rhs(st)
    c1["steps"].append({
        "step": step, "mass": s.quadrature_total(st, 0), "energy": s.quadrature_total(st, 4),
        "entropy": s.total_entropy(st), "production": s.entropy_production(st, rhs),
        "rhs3_max_abs": float(np.abs(rhs[:, 3]).max()), "q_max_abs": [float(np.abs(st[:, v]).max()) for v in range(5)],
        "q_fnv": "%016x" % po.fnv1a64(st)})
    if step < 10:
        s.step(dt)
kats["config1_bubble_sharp_L3_N4_f64"] = c1
# a thin slab of the 10-step state (elements 0..15) as a spot check
arrays["config1_state10_elems0_16"] = s.state[:16].copy()

# --- EntropyTestState seed 20240501, bubble_mesh(1, periodic z), N=4 --------
for diss in (False, True):
    s = R.mesh(po.bubble_mesh_config(1, True)).solver(4, "f64", settings=po.make_settings(diss))
    q = s.init_case(po.CASE_ENTROPY_TEST, 20240501).copy()
    rhs = s.assemble_rhs(q)
    tag = "diss" if diss else "ec"
    arrays["entropy_q"] = q
    arrays[f"entropy_rhs_{tag}"] = rhs
    kats[f"entropy_test_20240501_{tag}"] = {
        "rhs_max_abs": [float(np.abs(rhs[:, v]).max()) for v in range(5)],
        "entropy": s.total_entropy(q), "production": s.entropy_production(q, rhs),
        "rhs_fnv": "%016x" % po.fnv1a64(rhs)}
arrays["entropy_volume_rhs"] = s.volume_rhs(q)

# --- FP32 of the same state ------------------------------------------------------
s = R.mesh(po.bubble_mesh_config(1, True)).solver(4, "f32")
q32 = s.init_case(po.CASE_ENTROPY_TEST, 20240501).copy()
arrays["entropy_q_f32"] = q32
arrays["entropy_rhs_diss_f32"] = s.assemble_rhs(q32)

# --- partitioned trajectory (test_partition.cpp:76-100): order 3, 10 steps --
s = R.mesh(po.bubble_mesh_config(1, False)).solver(3, "f64", ranks=2)
s.init_case(po.CASE_BUBBLE_SHARP)
dt3 = s.compute_dt(0.5)
for _ in range(10):
    s.step(dt3)
arrays["bubble_L1_N3_state10"] = s.state.copy()
kats["bubble_L1_N3"] = {"dt": dt3}

# --- beta-plane Coriolis on a small channel ----------------------------------------
cfg = po.mesh_config((2, 1, 1), 1, (0., 0., 0.), (4e6, 6e6, 3e4), (0, 1, 1))
s = R.mesh(cfg).solver(3, "f64", settings=po.make_settings(True, 2, 1e-4, 1.6e-11, 3e6))
q = s.init_case(po.CASE_ENTROPY_TEST, 13).copy()
arrays["coriolis_q"] = q
arrays["coriolis_rhs"] = s.assemble_rhs(q)

# --- operators ----------------------------------------------------------------------
for order in (1, 2, 3, 4, 5, 6, 7):
    x, w, d = R.reference_element(order)
    arrays[f"lgl_nodes_{order}"], arrays[f"lgl_weights_{order}"], arrays[f"lgl_diff_{order}"] = x, w, d
a, b, c = R.lsrk()
arrays["lsrk_a"], arrays["lsrk_b"], arrays["lsrk_c"] = a, b, c

# --- pointwise physics KATs (reference's tests/test_physics.cpp:139-168) -----------
def vals(s64, rho, u, p, phi):
    q5 = np.array([rho, rho * u[0], rho * u[1], rho * u[2],
                   p / 0.4 + 0.5 * rho * sum(x * x for x in u) + rho * phi])
    rc, nv = s64.node_vals(q5, phi)
    assert rc == 0
    return nv
s64 = R.mesh(po.unit_mesh_config(0)).solver(1, "f64")
m = vals(s64, 1.0, (0, 0, 0), 1e5, 0.0)
p = vals(s64, 2.0, (0, 0, 0), 1e5, 9.81)
kats["rho_hat_example_flux"] = [float(x) for x in s64.ec_flux(m, p, 0)]
v = vals(s64, 1.0, (2.0, 0, 0), 1e5, 0.0)
kats["spec_consistency_flux"] = [float(x) for x in s64.ec_flux(v, v, 0)]
rng = np.random.default_rng(20240815)
pairs = []
for _ in range(64):
    a8 = vals(s64, rng.uniform(0.5, 2.0), rng.uniform(-50, 50, 3), rng.uniform(5e4, 2e5), rng.uniform(0, 2e4))
    b8 = vals(s64, rng.uniform(0.5, 2.0), rng.uniform(-50, 50, 3), rng.uniform(5e4, 2e5), rng.uniform(0, 2e4))
    d = int(rng.integers(0, 3))
    pairs.append(np.concatenate([a8, b8, [d], s64.ec_flux(a8, b8, d), s64.matrix_dissipation(a8, b8, d)]))
arrays["pointwise_pairs"] = np.array(pairs)   # 8 + 8 + 1 + 7 + 5 columns

np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
with open(os.path.join(HERE, "kats.json"), "w") as f:
    json.dump(kats, f, indent=1)
print("wrote", len(arrays), "arrays;", os.path.getsize(os.path.join(HERE, "golden.npz")), "bytes")
