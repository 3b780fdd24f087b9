"""GPU parity of the nested Bregman loop through the C ABI against the CPU
oracle and the dense Kronecker oracle (test_solver.cpp:179-365,
acceptance.cpp:43-92; north_star parity gates)."""
import numpy as np
import pytest

import oracle as O
from conftest import random_graph
from dense_oracles import KroneckerSolver, diff_matrix_dense
from paper_1612_06496_b200 import api
from paper_1612_06496_b200.inputs import grid_graph, knn_graph, make_config, voronoi_image

pytestmark = pytest.mark.gpu


def jacobi(d, lam=1.0, r=1.0, soc=3, sb=4, tol=1e-6, maxit=50, stage2=0, conv=0.0):
    return api.PfeParams(dim=d, lambda_=lam, r=r, soc_max=soc, sb_max_stage1=sb, sb_max_stage2=stage2,
                         conv_tol=conv, pcg=api.PcgConfig(tol, maxit, api.Preconditioner.Jacobi))


def rel_fro_signed(a, b):
    """||A - B||_F / ||B||_F after per-column sign alignment (north_star gate)."""
    s = np.sign(np.sum(a * b, axis=0))
    s[s == 0] = 1.0
    return np.linalg.norm(a * s - b) / np.linalg.norm(b)


def label_agreement(a, b):
    """Best label matching through the contingency table (Hungarian)."""
    from scipy.optimize import linear_sum_assignment

    ka, kb = a.max() + 1, b.max() + 1
    t = np.zeros((ka, kb), np.int64)
    np.add.at(t, (a, b), 1)
    r, c = linear_sum_assignment(-t)
    return t[r, c].sum() / a.size


def test_single_edge_hand_rolled():
    # test_solver.cpp:194-219
    g = api.WeightedGraph(2, [0], [1], [1.0], [1.0, 1.0])
    lam, r = 2.0, 1.0
    p = np.array([[1.0], [-1.0]])
    sys_ = np.array([[lam / 2 + r / 2, -lam / 2], [-lam / 2, lam / 2 + r / 2]])
    y_hand = np.linalg.solve(sys_, np.array([r / 2, -r / 2]))
    traj = []
    prm = api.PfeParams(dim=1, lambda_=lam, r=r, conv_tol=0.0, pcg=api.PcgConfig(1e-13, 2000))
    api.split_bregman(g, g.degree, p, np.zeros((2, 1)), prm, np.zeros((2, 1)), 1,
                      on_iterate=lambda it, y: traj.append(y))
    assert len(traj) == 1
    assert np.abs(traj[0][:, 0] - y_hand).max() < 1e-10


def test_quadratic_limit():
    # test_solver.cpp:179-192
    rng = np.random.Generator(np.random.PCG64(23))
    g = random_graph(8, 8, rng)
    p, b = rng.uniform(-1, 1, (8, 2)), rng.uniform(-1, 1, (8, 2))
    prm = api.PfeParams(dim=2, lambda_=1e-12, r=1.0, conv_tol=0.0, pcg=api.PcgConfig(1e-13, 2000))
    y = api.split_bregman(g, g.degree, p, b, prm, np.zeros((8, 2)), 1)
    assert np.abs(y - np.diag(1 / np.sqrt(g.degree)) @ (p - b)).max() < 1e-6


def test_trajectory_matches_kronecker_acceptance_1():
    """Acceptance criterion 1: 25 tiny instances, 8 SB iterations, <= 1e-8."""
    rng = np.random.Generator(np.random.PCG64(101))
    worst = 0.0
    for _ in range(25):
        n, d = int(rng.integers(3, 7)), int(rng.integers(1, 4))
        g = random_graph(n, 2, rng)
        y0, p, b = rng.normal(size=(n, d)), rng.normal(size=(n, d)), 0.2 * rng.normal(size=(n, d))
        prm = api.PfeParams(dim=d, lambda_=50.0, r=1.5, conv_tol=0.0, pcg=api.PcgConfig(1e-13, 10000))
        got = []
        api.split_bregman(g, g.degree, p, b, prm, y0, 8, on_iterate=lambda it, y: got.append(y))
        lit = []
        KroneckerSolver(diff_matrix_dense(g), g.degree, d, 50.0, 1.5).split_bregman(p, b, y0, 8, lit)
        assert len(got) == 8
        worst = max(worst, max(np.abs(a - c).max() for a, c in zip(got, lit)))
    assert worst <= 1e-8


def test_trajectory_matches_oracle_jacobi():
    """Same Jacobi-PCG on both sides: only reduction order differs."""
    rng = np.random.Generator(np.random.PCG64(29))
    for _ in range(10):
        n, d = int(rng.integers(20, 60)), int(rng.integers(1, 6))
        g = random_graph(n, 2 * n, rng)
        y0, p, b = rng.normal(size=(n, d)), rng.normal(size=(n, d)), 0.3 * rng.normal(size=(n, d))
        prm = jacobi(d, lam=8.0, r=1.5, tol=1e-8, maxit=200)
        got = []
        api.split_bregman(g, g.degree, p, b, prm, y0, 6, on_iterate=lambda it, y: got.append(y))
        _, exp = O.split_bregman(g, g.degree, p, b, prm, y0, 6, want_traj=True)
        for a, c in zip(got, exp):
            assert np.abs(a - c).max() <= 1e-11 * max(1.0, np.abs(c).max())


def test_soc_matches_literal_outer_loop():
    # test_solver.cpp:252-271 (IC0 params -> Jacobi on the GPU, tight tolerance)
    rng = np.random.Generator(np.random.PCG64(31))
    for trial in range(5):
        g = random_graph(6, 4, rng)
        y0 = api.random_embedding(6, 2, trial, g.degree)
        exp = KroneckerSolver(diff_matrix_dense(g), g.degree, 2, 10.0, 1.0).soc(y0, 3, 4)
        prm = api.PfeParams(dim=2, lambda_=10.0, r=1.0, soc_max=3, sb_max_stage1=4, conv_tol=0.0,
                            pcg=api.PcgConfig(1e-13, 2000))
        got = api.soc(g, prm, y0)
        assert np.abs(got - exp).max() < 1e-7


@pytest.mark.parametrize("use_graphs", [True, False])
def test_soc_random_graphs_match_oracle(use_graphs):
    rng = np.random.Generator(np.random.PCG64(77))
    for d in [1, 2, 3, 5, 8, 16]:
        n = 300
        g = random_graph(n, 3 * n, rng)
        prm = jacobi(d, soc=3, sb=5)
        y0 = api.random_embedding(n, d, d, g.degree)
        got = api.soc(g, prm, y0, use_graphs=use_graphs)
        exp = O.solve(g, prm, y0, mode=0)
        assert rel_fro_signed(got, exp) <= 1e-10, d


def test_keeps_split_variable_orthonormal():
    # test_solver.cpp:273-286
    rng = np.random.Generator(np.random.PCG64(37))
    g = random_graph(12, 14, rng)
    prm = api.PfeParams(dim=3, soc_max=4, sb_max_stage1=3, pcg=api.PcgConfig(1e-6, 1000))
    s = api.PfeSolver(g, prm, warn=False)
    st = s.make_state(api.random_embedding(12, 3, 1, g.degree))
    s.run_soc(st, 4, 3)
    p = st.p
    assert np.abs(p.T @ p - np.eye(3)).max() < 1e-8


def small_image(h=40, w=60, seed=3, radius=1, sigma_xy=None):
    rng = np.random.Generator(np.random.PCG64(seed))
    img, _ = voronoi_image(h, w, 5, 0.05, rng)
    return grid_graph(img, 0.1 if radius == 1 else 0.1, radius, sigma_xy)


@pytest.mark.parametrize("radius,sxy", [(1, None), (2, 2.0)])
def test_grid_stencil_path_matches_oracle(radius, sxy):
    g = small_image(radius=radius, sigma_xy=sxy)
    for d in [3, 4, 8]:
        prm = jacobi(d, soc=3, sb=6)
        s = api.PfeSolver(g, prm, warn=False)
        assert s.report()["topology"] == radius  # stencil kernels in use
        y0 = api.random_embedding(g.n, d, 11, g.degree)
        st = s.make_state(y0)
        s.run_soc(st, 3, 6)
        exp = O.solve(g, prm, y0, mode=0, full_state=True)
        assert rel_fro_signed(st.y, exp["y"]) <= 1e-10
        assert np.abs(st.bregman - exp["bregman"]).max() <= 1e-9
        assert np.abs(st.split_b - exp["split_b"]).max() <= 1e-9
        assert np.abs(st.split_s - exp["split_s"]).max() <= 1e-9


def test_grid_and_csr_paths_agree_bitwise():
    g = small_image()
    prm = jacobi(4, soc=2, sb=5)
    y0 = api.random_embedding(g.n, 4, 1, g.degree)
    a = api.soc(g, prm, y0)
    g2 = api.WeightedGraph(g.n, g.ei, g.ej, g.w, g.degree)  # no grid hint -> CSR kernels
    b = api.soc(g2, prm, y0)
    # identical per-vertex arithmetic; only the grid size of the reductions differs
    assert rel_fro_signed(a, b) <= 1e-13


def test_graph_and_host_driven_agree_bitwise():
    g = small_image()
    prm = jacobi(4, soc=3, sb=5)
    y0 = api.random_embedding(g.n, 4, 2, g.degree)
    a = api.soc(g, prm, y0, use_graphs=True, persistent=False)
    b = api.soc(g, prm, y0, use_graphs=False, persistent=False)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("kind", ["resident", "tiled"])
@pytest.mark.parametrize("radius,d", [(1, 4), (1, 8), (1, 3), (2, 8), (2, 2)])
def test_persistent_kernel_matches_multi_kernel_path(radius, d, kind):
    """The cooperative persistent split-Bregman kernels (state resident in
    shared memory, or tiles streamed from L2/HBM) compute the same
    per-element arithmetic as the one-kernel-per-phase path; only the
    reduction trees (grid sizes) differ."""
    g = small_image(48, 70, seed=5, radius=radius, sigma_xy=2.0 if radius == 2 else None)
    prm = jacobi(d, soc=3, sb=6)
    y0 = api.random_embedding(g.n, d, 4, g.degree)
    mode = True if kind == "resident" else "tiled"
    s = api.PfeSolver(g, prm, warn=False, persistent=mode)
    st = s.make_state(y0)
    s.run_soc(st, prm.soc_max, prm.sb_max_stage1)
    a = st.y
    assert s.report()["persistent_kind"] == (2 if kind == "resident" else 1)
    b = api.soc(g, prm, y0, persistent=False)
    assert rel_fro_signed(a, b) <= 1e-12
    exp = O.solve(g, prm, y0, mode=0)
    assert rel_fro_signed(a, exp) <= 1e-10
    # state after a persistent call is complete (split_s materialised)
    s = api.PfeSolver(g, prm, warn=False, persistent=mode)
    st = s.make_state(y0)
    s.run_soc(st, 2, 4)
    full = O.solve(g, jacobi(d, soc=2, sb=4), y0, mode=0, full_state=True)
    assert np.abs(st.split_s - full["split_s"]).max() <= 1e-9
    assert np.abs(st.split_b - full["split_b"]).max() <= 1e-9


@pytest.mark.parametrize("h,w,radius,d", [(33, 70, 2, 8), (21, 64, 2, 4), (47, 38, 2, 2), (30, 71, 2, 4), (40, 66, 1, 4),
                                          (37, 70, 1, 8), (31, 65, 1, 2), (9, 40, 1, 4)])
def test_tiled_persistent_tma_staging_bitwise(h, w, radius, d, monkeypatch):
    """The tiled persistent kernel stages 5x5-grid tiles with TMA boxes (even
    d and width) and 8-neighbour tiles with cp.async.bulk row copies (even
    d), else per-element cp.async (PFE_TMA=0 PFE_BULK=0): staging must not
    change a single bit; ragged and border tiles are zero-filled by all."""
    g = small_image(h, w, seed=h * w, radius=radius, sigma_xy=2.0 if radius == 2 else None)
    prm = jacobi(d, soc=2, sb=5)
    y0 = api.random_embedding(g.n, d, 2, g.degree)
    out = {}
    # staging variants: TMA boxes (5x5 default; every phase for 8-neighbour
    # grids with PFE_TMA=1, whose inv-diag halo stays on cp.async), bulk row
    # copies (PFE_BULK=1, when TMA is off), per-element cp.async
    variants = {"tma": {"PFE_TMA": "1", "PFE_BULK": "0"}, "bulk": {"PFE_TMA": "0", "PFE_BULK": "1"},
                "cpasync": {"PFE_TMA": "0", "PFE_BULK": "0"}}
    for name, env in variants.items():
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        s = api.PfeSolver(g, prm, warn=False, persistent="tiled")
        st = s.make_state(y0)
        s.run_soc(st, prm.soc_max, prm.sb_max_stage1)
        assert s.report()["persistent_kind"] == 1
        out[name] = (st.y, st.split_b, st.split_s)
    for name in ("tma", "bulk"):
        for a, b in zip(out[name], out["cpasync"]):
            assert np.array_equal(a, b), name
    exp = O.solve(g, prm, y0, mode=0)
    assert rel_fro_signed(out["tma"][0], exp) <= 1e-10


@pytest.mark.parametrize("h,w,radius,d", [(1, 200, 1, 4), (300, 4, 1, 4), (5, 300, 2, 4), (17, 6, 2, 2),
                                            (150, 151, 1, 4), (3, 4, 1, 1)])
def test_resident_kernel_region_shapes(h, w, radius, d):
    """Region grids with 1-pixel-wide regions, regions thinner than the ring,
    images smaller than the region count: same result as the multi-kernel path."""
    g = small_image(h, w, seed=h + w, radius=radius, sigma_xy=2.0 if radius == 2 else None)
    prm = jacobi(d, soc=2, sb=4)
    y0 = api.random_embedding(g.n, d, 6, g.degree)
    s = api.PfeSolver(g, prm, warn=False)
    st = s.make_state(y0)
    s.run_soc(st, 2, 4)
    assert s.report()["persistent_kind"] == 2
    b = api.soc(g, prm, y0, persistent=False)
    assert rel_fro_signed(st.y, b) <= 1e-12


def test_resident_kernel_with_callback_and_conv_tol():
    """One launch per inner iteration (callback / relative-change test): the
    rhs handed from launch to launch keeps the iteration identical."""
    g = small_image(60, 80, seed=9)
    prm = jacobi(4, soc=2, sb=5)
    y0 = api.random_embedding(g.n, 4, 3, g.degree)
    p, b0 = y0, 0.1 * y0
    seen = []
    a = api.split_bregman(g, g.degree, p, b0, prm, y0 * 0.5, 5, on_iterate=lambda it, y: seen.append(it))
    b = api.split_bregman(g, g.degree, p, b0, prm, y0 * 0.5, 5, persistent=False)
    assert seen == list(range(5))
    assert rel_fro_signed(a, b) <= 1e-12


def test_state_outliving_its_solver_is_safe():
    """Destroying a solver before its state (Python GC order) must not break
    later solvers: states return their memory to the pool independently."""
    g = small_image(30, 40, seed=4)
    prm = jacobi(4, soc=2, sb=3)
    y0 = api.random_embedding(g.n, 4, 2, g.degree)
    s = api.PfeSolver(g, prm, warn=False)
    st = s.make_state(y0)
    s.run_soc(st, 2, 3)
    s.close()
    del st
    for _ in range(3):
        s2 = api.PfeSolver(g, prm, warn=False)
        st2 = s2.make_state(y0)
        s2.run_soc(st2, 2, 3)
        y = st2.y
        s2.close()
    assert rel_fro_signed(y, api.soc(g, prm, y0, persistent=False)) <= 1e-12


def test_deterministic_runs():
    # test_solver.cpp:353-365
    rng = np.random.Generator(np.random.PCG64(41))
    g = random_graph(10, 12, rng)
    prm = api.PfeParams(dim=2, soc_max=3, sb_max_stage1=3, sb_max_stage2=10, pcg=api.PcgConfig(1e-6, 1000))
    y0 = api.random_embedding(10, 2, 9, g.degree)
    assert np.array_equal(api.pfe_two_stage(g, prm, y0), api.pfe_two_stage(g, prm, y0))
    s = api.PfeSolver(g, jacobi(2), warn=False)
    st = s.make_state(y0)
    s.run_soc(st, 2, 3)
    y1 = st.y
    st.reset()
    s.run_soc(st, 2, 3)
    assert np.array_equal(y1, st.y)


def test_two_stage_with_stage2_and_conv_tol_matches_oracle():
    g = small_image(30, 40, seed=8)
    for conv in [0.0, 1e-4]:
        prm = jacobi(4, soc=4, sb=5, stage2=12, conv=conv)
        y0 = api.random_embedding(g.n, 4, 3, g.degree)
        got = api.pfe_two_stage(g, prm, y0)
        exp = O.solve(g, prm, y0, mode=1)
        assert rel_fro_signed(got, exp) <= 1e-9
        # stage II disabled reproduces stage I exactly (test_solver.cpp:300-306)
        prm.sb_max_stage2 = 0
        assert np.array_equal(api.pfe_two_stage(g, prm, y0), api.soc(g, prm, y0))


def test_state_roundtrip_and_split_bregman_on_state():
    g = small_image(20, 30, seed=4)
    d = 3
    prm = jacobi(d, lam=2.0, r=0.7)
    s = api.PfeSolver(g, prm, warn=False)
    y0 = api.random_embedding(g.n, d, 5, g.degree)
    st = s.make_state(y0)
    assert np.array_equal(st.y, y0)
    assert np.array_equal(st.p, np.sqrt(g.degree)[:, None] * y0)
    assert not st.bregman.any() and not st.split_b.any() and not st.split_s.any()
    rng = np.random.Generator(np.random.PCG64(6))
    vals = {k: rng.normal(size=(g.n if k in ("p", "bregman") else g.m, d)) * 0.3 for k in
            ("p", "bregman", "split_b", "split_s")}
    for k, v in vals.items():
        setattr(st, k, v)
        assert np.array_equal(getattr(st, k), v)
    traj = []
    s.split_bregman(st, 4, on_iterate=lambda it, y: traj.append(y))
    exp = O.state_split_bregman(g, prm, 4, y0, vals["p"], vals["bregman"], vals["split_b"], vals["split_s"],
                                want_traj=True)
    assert len(traj) == 4
    for a, c in zip(traj, exp["traj"]):
        assert np.abs(a - c).max() <= 1e-11
    for k in ("y", "p", "bregman", "split_b", "split_s"):
        assert np.abs(getattr(st, k) - exp[k]).max() <= 1e-10, k


def record_parity(name, g, prm, y, exp, pcg_gpu, pcg_oracle, k):
    """Measured parity of a full-size configuration against the oracle
    (north_star gates), printed and written to gpurun_out/full_parity_<name>.json."""
    import json
    from pathlib import Path

    err = rel_fro_signed(y, exp)
    o1, o2 = api.objective(g, y), O.objective(g, exp)
    agree = label_agreement(api.kmeans(y, k, 0), O.kmeans(exp, k, 0))
    mism = int(np.sum(np.asarray(pcg_gpu) != np.asarray(pcg_oracle)))
    rec = {"config": name, "n": g.n, "m": g.m, "d": prm.dim, "inner": int(len(pcg_oracle)),
           "rel_err": {"fro": err, "objective": abs(o1 - o2) / abs(o2)}, "objective_gpu": o1,
           "objective_oracle": o2, "label_agreement": agree, "pcg_log_mismatches": mism,
           "pcg_iterations_gpu": int(np.sum(pcg_gpu)), "pcg_iterations_oracle": int(np.sum(pcg_oracle))}
    print(json.dumps(rec))
    out = Path(__file__).resolve().parents[1] / "gpurun_out"
    out.mkdir(exist_ok=True)
    (out / f"full_parity_{name}.json").write_text(json.dumps(rec, indent=1))
    assert err <= 1e-6
    assert abs(o1 - o2) <= 1e-6 * abs(o2)
    assert agree >= 0.999
    return rec


def test_knn_c1_full_size_parity():
    """BASELINE config C1 at full size: Y, objective, labels and the PCG log
    vs the oracle."""
    cfg = make_config("c1")
    g, prm = cfg.graph, cfg.params
    y0 = api.random_embedding(g.n, prm.dim, cfg.y0_seed, g.degree)
    s = api.PfeSolver(g, prm, warn=False)
    st = s.make_state(y0)
    s.run_soc(st, prm.soc_max, prm.sb_max_stage1)
    y = st.y
    its, _, _ = s.pcg_log()
    res = O.solve(g, prm, y0, mode=0, log_cap=1000)
    rec = record_parity("c1", g, prm, y, res["y"], its.max(axis=1), res["pcg_log"], cfg.k)
    assert rec["pcg_log_mismatches"] == 0


@pytest.mark.slow
def test_c2_full_size_parity():
    """BASELINE config C2 (481x321, d=4, 10x20, Jacobi tol 1e-6) vs the oracle:
    Y, objective, labels and the PCG log."""
    cfg = make_config("c2")
    g, prm = cfg.graph, cfg.params
    y0 = api.random_embedding(g.n, prm.dim, cfg.y0_seed, g.degree)
    s = api.PfeSolver(g, prm, warn=False)
    st = s.make_state(y0)
    s.run_soc(st, prm.soc_max, prm.sb_max_stage1)
    got = st.y
    its, _, _ = s.pcg_log()
    O.set_threads(4)
    try:
        res = O.solve(g, prm, y0, mode=0, log_cap=1000)
    finally:
        O.set_threads(1)
    rec = record_parity("c2", g, prm, got, res["y"], its.max(axis=1), res["pcg_log"], cfg.k)
    assert rec["pcg_log_mismatches"] == 0


def test_pcg_iteration_log_matches_oracle():
    g = small_image(30, 40, seed=9)
    prm = jacobi(4, soc=2, sb=5)
    y0 = api.random_embedding(g.n, 4, 1, g.degree)
    s = api.PfeSolver(g, prm, warn=False)
    st = s.make_state(y0)
    s.run_soc(st, 2, 5)
    its, status, rel = s.pcg_log()
    exp = O.solve(g, prm, y0, mode=0, log_cap=100)
    assert list(its.max(axis=1)) == list(exp["pcg_log"])
    rep = s.report()
    assert rep["inner_iterations"] == 10 and rep["pcg_iterations"] == int(exp["pcg_log"].sum())
