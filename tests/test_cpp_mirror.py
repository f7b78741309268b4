"""The header-only C++ mirror of the reference interface
(include/esdg_b200/gpu_solver.hpp): compiles everywhere, runs on a GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2605_16684_b200", "csrc")
ORACLE = os.path.join(ROOT, "oracle")
REF = "/root/reference/proj/core/include"


def _build(tmp_path):
    exe = tmp_path / "test_gpu_solver"
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), "-I", ORACLE,
                    os.path.join(ROOT, "tests", "cpp", "test_gpu_solver.cpp"), "-o", str(exe),
                    "-L", CSRC, "-lesdg_b200", "-L", ORACLE, "-loracle",
                    f"-Wl,-rpath,{CSRC}", f"-Wl,-rpath,{ORACLE}"], check=True)
    return exe


def test_cpp_mirror_compiles(tmp_path, port):
    _build(tmp_path)


def test_cpp_mirror_compiles_against_reference_types(tmp_path):
    """With ESDG_B200_WITH_REFERENCE the header takes the reference's own
    MeshGeometry / GasConstants / KernelSettings and throws its exception."""
    if not os.path.isdir(REF):
        pytest.skip("reference tree not present")
    src = tmp_path / "with_ref.cpp"
    src.write_text("""
        #define ESDG_B200_WITH_REFERENCE
        #include "esdg_b200/gpu_solver.hpp"
        #include "esdg/state.hpp"
        double f(std::shared_ptr<const esdg::MeshGeometry> mesh) {
          esdg::KernelSettings<double> s;
          esdg_b200::GpuSolver<double> solver(mesh, 4, esdg::GasConstants<double>{}, s, 1);
          esdg::StateField<double> q(mesh->num_elements(), solver.n3()), out(mesh->num_elements(), solver.n3());
          try { solver.assemble_rhs(q, out, 0.0, 1.0); solver.step(1e-3); }
          catch (const esdg::NonPhysicalState& e) { return e.rho(); }
          return solver.compute_dt(0.5);
        }
    """)
    subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"), "-I", REF,
                    str(src)], check=True)


@pytest.mark.gpu
def test_cpp_mirror_runs(tmp_path, port):
    exe = _build(tmp_path)
    res = subprocess.run([str(exe)], capture_output=True, text=True)
    print(res.stdout, res.stderr)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "ALL PASSED" in res.stdout
