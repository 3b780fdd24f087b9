"""The link-level backend (paper_1612_06496_b200/binding/pfe_core_b200.cpp)
behind the reference's OWN headers.

tests/cpp/test_ref_binding.cpp includes /root/reference/proj/core/include/
pfe/{solver,pcg,graph,errors}.hpp, calls pfe::soc, pfe::PfeSolver
(make_state / run_soc / split_bregman with an IterateCallback),
pfe::pfe_two_stage (the call tools/main.cpp:121 makes), pfe::objective and
pfe::PcgOperator / pcg_solve_multi, and is linked against the binding and
libpfe_b200.so (build.py: build_ref_binding).  The binary is built in the
build container (it needs the reference's headers) and travels to the GPU box.

* CPU: every symbol solver.cpp / pcg.cpp define is defined by the binding,
  and without a device the reference API raises pfe::ConfigError (exit 3,
  the CLI mapping main.cpp:431-446) -- no CPU fallback.
* GPU: the outputs match the CPU oracle on a golden fixture.
"""
import os
import struct
import subprocess
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from golden.make_golden import load
from paper_1612_06496_b200 import build as B

ROOT = Path(__file__).resolve().parents[1]
BIN = B.REF_TEST
SRC = ROOT / "paper_1612_06496_b200" / "binding" / "pfe_core_b200.cpp"


def _bin():
    if not BIN.exists():
        if B.REF_INCLUDE.exists() and B.LIB.exists():
            B.build_ref_binding()
        else:
            pytest.skip("test_ref_binding not built (needs /root/reference headers in the build container)")
    return BIN


def spd_matrix(n=40, seed=3):
    """Symmetric diagonally dominant tridiagonal-plus CSR (rows sorted)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    a = np.zeros((n, n))
    for i in range(n):
        for j in (i - 3, i - 1, i + 1, i + 3):
            if 0 <= j < n:
                a[i, j] = a[j, i] = -rng.uniform(0.1, 1.0)
    a[np.arange(n), np.arange(n)] = np.abs(a).sum(1) + 0.5
    ptr, idx, val = [0], [], []
    for i in range(n):
        nz = np.nonzero(a[i])[0]
        idx += list(nz)
        val += list(a[i, nz])
        ptr.append(len(idx))
    return np.array(ptr, np.int32), np.array(idx, np.int32), np.array(val), a


def write_input(path, g, prm, y0, a, b, x0):
    ptr, idx, val = a
    with open(path, "wb") as f:
        f.write(struct.pack("<8i", g.n, g.m, prm.dim, prm.soc_max, prm.sb_max_stage1, prm.sb_max_stage2,
                            prm.pcg.max_iter, int(prm.pcg.preconditioner)))
        f.write(struct.pack("<4d", prm.lambda_, prm.r, prm.conv_tol, prm.pcg.rel_tol))
        for arr, dt in ((g.ei, np.int32), (g.ej, np.int32), (g.w, np.float64), (g.degree, np.float64)):
            f.write(np.ascontiguousarray(arr, dt).tobytes())
        f.write(np.asfortranarray(y0).tobytes(order="F"))
        f.write(struct.pack("<2i", len(ptr) - 1, len(val)))
        f.write(ptr.tobytes() + idx.tobytes() + val.tobytes())
        f.write(np.asfortranarray(b).tobytes(order="F") + np.asfortranarray(x0).tobytes(order="F"))


def read_output(path, n, d, an):
    raw = Path(path).read_bytes()
    off = 0

    def take(count, dt):
        nonlocal off
        arr = np.frombuffer(raw, dt, count, off)
        off += arr.nbytes
        return arr

    nd = n * d
    out = {k: take(nd, np.float64).reshape(d, n).T for k in ("soc", "state", "two_stage", "cb")}
    out["objective"], out["callbacks"] = take(2, np.float64)
    out["pcg_x"] = take(an * 2, np.float64).reshape(2, an).T
    out["pcg_iters"] = take(2, np.int32)
    out["vec_x"] = take(an, np.float64)
    out["vec_iters"] = int(take(1, np.int32)[0])
    out["fallback"] = int(take(1, np.int32)[0])
    return out


def case(tmp_path):
    g, prm, mode, k, z = load(ROOT / "tests" / "golden" / "grid8_c2like.npz")
    prm.sb_max_stage2 = 3
    a = spd_matrix()
    rng = np.random.Generator(np.random.PCG64(9))
    b = rng.normal(size=(len(a[0]) - 1, 2))
    x0 = np.zeros_like(b)
    fin = tmp_path / "in.bin"
    write_input(fin, g, prm, z["y0"], a[:3], b, x0)
    return g, prm, z, a, b, x0, fin


def test_binding_defines_every_solver_and_pcg_symbol():
    """Every out-of-line function of the reference's solver.hpp / pcg.hpp
    (solver.cpp / pcg.cpp definitions) is defined by the binding."""
    if not B.REF_INCLUDE.exists():
        pytest.skip("needs /root/reference headers")
    obj = Path(os.environ.get("TMPDIR", "/tmp")) / "pfe_core_b200_symcheck.o"
    subprocess.run(["g++", "-std=c++20", "-O0", "-c", f"-I{B.EIGEN_STUB}", f"-I{B.REF_INCLUDE}", f"-I{B.INCLUDE}",
                    str(SRC), "-o", str(obj)], check=True)
    syms = subprocess.run(["nm", "-C", "--defined-only", str(obj)], capture_output=True, text=True,
                          check=True).stdout
    need = ["pfe::objective(pfe::CsrMatrix const&, Eigen::MatrixXd const&)",
            "pfe::shrink(Eigen::MatrixXd const&, double)",
            "pfe::project_orthogonal(Eigen::MatrixXd const&)",
            "pfe::PfeSolver::PfeSolver(pfe::WeightedGraph const&, pfe::PfeParams const&)",
            "pfe::PfeSolver::split_bregman(pfe::SolverState&, int, std::function<void (int, Eigen::MatrixXd const&)> const&) const",
            "pfe::PfeSolver::run_soc(pfe::SolverState&, int, int) const",
            "pfe::PfeSolver::two_stage(Eigen::MatrixXd const&) const",
            "pfe::PfeSolver::make_state(Eigen::MatrixXd const&) const",
            "pfe::split_bregman(pfe::CsrMatrix const&, Eigen::VectorXd const&, Eigen::MatrixXd const&, "
            "Eigen::MatrixXd const&, pfe::PfeParams const&, Eigen::MatrixXd const&, int, "
            "std::function<void (int, Eigen::MatrixXd const&)> const&)",
            "pfe::soc(pfe::WeightedGraph const&, pfe::PfeParams const&, Eigen::MatrixXd const&)",
            "pfe::pfe_two_stage(pfe::WeightedGraph const&, pfe::PfeParams const&, Eigen::MatrixXd const&)",
            "pfe::save_embedding(Eigen::MatrixXd const&, std::__cxx11::basic_string<char, std::char_traits<char>, std::allocator<char> > const&)",
            "pfe::load_embedding(std::__cxx11::basic_string<char, std::char_traits<char>, std::allocator<char> > const&)",
            "pfe::PcgOperator::PcgOperator(pfe::CsrMatrix, pfe::PcgConfig)",
            "pfe::PcgOperator::solve(Eigen::VectorXd const&, Eigen::VectorXd const&) const",
            "pfe::PcgOperator::solve_multi(Eigen::MatrixXd const&, Eigen::MatrixXd const&) const",
            "pfe::pcg_solve(pfe::CsrMatrix const&, Eigen::VectorXd const&, Eigen::VectorXd const&, pfe::PcgConfig const&)",
            "pfe::pcg_solve_multi(pfe::CsrMatrix const&, Eigen::MatrixXd const&, Eigen::MatrixXd const&, pfe::PcgConfig const&)"]
    missing = [s for s in need if s not in syms]
    assert not missing, missing


def test_reference_api_without_device_raises_config_error(tmp_path):
    from paper_1612_06496_b200 import _native as N

    if N.load().pfe_device_check(0) == 0:
        pytest.skip("a device is present: covered by the GPU test")
    _, _, _, _, _, _, fin = case(tmp_path)
    r = subprocess.run([str(_bin()), str(fin), str(tmp_path / "out.bin")], capture_output=True, text=True)
    assert r.returncode == 3, r.stdout + r.stderr
    assert r.stdout.startswith("ConfigError:")


@pytest.mark.gpu
def test_reference_api_on_gpu_matches_oracle(tmp_path):
    g, prm, z, a, b, x0, fin = case(tmp_path)
    fout = tmp_path / "out.bin"
    r = subprocess.run([str(_bin()), str(fin), str(fout)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "expected ConfigError: PfeSolver: dim must be >= 1" in r.stdout
    out = read_output(fout, g.n, prm.dim, len(a[0]) - 1)
    exp = z["y"]  # oracle soc on this fixture (tests/golden/make_golden.py)
    err = np.linalg.norm(out["soc"] - exp) / np.linalg.norm(exp)
    assert err <= 1e-9
    assert np.array_equal(out["soc"], out["state"])  # PfeSolver path == one-call path, bitwise
    ts = O.solve(g, prm, z["y0"], mode=1)
    assert np.linalg.norm(out["two_stage"] - ts) / np.linalg.norm(ts) <= 1e-9
    assert out["callbacks"] == 3.0
    oo = O.objective(g, out["soc"])
    assert abs(out["objective"] - oo) <= 1e-12 * abs(oo)
    xe, its, _, _ = O.pcg_solve_multi(a[:3], b, x0, 1e-10, 200, 1)
    assert np.abs(out["pcg_x"] - xe).max() <= 1e-10 * np.abs(xe).max()
    assert list(out["pcg_iters"]) == list(its)
    assert np.abs(out["vec_x"] - xe[:, 0]).max() <= 1e-10 * np.abs(xe).max()
    assert out["fallback"] == 0
