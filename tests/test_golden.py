"""Committed golden fixtures (tests/golden/*.npz, made by tests/golden/make_golden.py).

CPU: the oracle re-derives every fixture exactly (pins the fixtures to the
oracle, which is itself pinned to the recorded reference run,
tests/test_oracle.py::test_golden_quadrant_run_matches_recorded_reference).
GPU: the CUDA path, called through the C ABI, meets the north_star parity
gates against the frozen numbers: rel. Frobenius error of Y <= 1e-6 up to
column sign, objective within 1e-6 relative, >= 99.9 % k-means label
agreement, and the same PCG iteration count in every inner iteration.
"""
import sys
from pathlib import Path

import numpy as np
import pytest

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE / "golden"))

import make_golden as MG  # noqa: E402

FIXTURES = sorted(p for p in (HERE / "golden").glob("*.npz") if not p.name.startswith("full_"))
IDS = [f.stem for f in FIXTURES]


def test_fixture_set_complete():
    assert set(IDS) == set(MG.cases()), "regenerate with python tests/golden/make_golden.py"


@pytest.mark.parametrize("path", FIXTURES, ids=IDS)
def test_oracle_reproduces_fixture(path):
    g, prm, mode, k, z = MG.load(path)
    got = MG.oracle_outputs(g, prm, int(z["iparams"][8]), mode, k)
    assert np.array_equal(got["y0"], z["y0"])
    assert np.abs(got["y"] - z["y"]).max() <= 1e-12 * max(1.0, np.abs(z["y"]).max())
    assert abs(got["objective"] - z["objective"]) <= 1e-12 * abs(z["objective"])
    assert np.array_equal(got["pcg_log"], z["pcg_log"])
    assert np.array_equal(got["labels"], z["labels"])


def test_fixture_inputs_regenerate():
    """The seeded input generators still produce the fixture graphs."""
    for path in FIXTURES:
        g, prm, mode, k, z = MG.load(path)
        g2, prm2, seed, mode2, k2 = MG.cases()[path.stem]
        assert g2.n == g.n and np.array_equal(g2.ei, g.ei) and np.array_equal(g2.ej, g.ej)
        assert np.array_equal(g2.w, g.w) and np.array_equal(g2.degree, g.degree)
        assert (prm2.dim, prm2.soc_max, prm2.sb_max_stage1, mode2, k2) == (prm.dim, prm.soc_max,
                                                                           prm.sb_max_stage1, mode, k)


@pytest.mark.gpu
@pytest.mark.parametrize("path", FIXTURES, ids=IDS)
def test_gpu_matches_fixture(path):
    from paper_1612_06496_b200 import api
    from test_gpu_solver import label_agreement, rel_fro_signed

    g, prm, mode, k, z = MG.load(path)
    s = api.PfeSolver(g, prm, warn=False)
    if mode == 0:
        st = s.make_state(z["y0"])
        s.run_soc(st, prm.soc_max, prm.sb_max_stage1)
    else:
        st = s.two_stage(z["y0"])
    y = st.y
    its, _, _ = s.pcg_log()
    # north_star gates (tolerances as stated there)
    assert rel_fro_signed(y, z["y"]) <= 1e-6
    obj = api.objective(g, y)
    assert abs(obj - z["objective"]) <= 1e-6 * abs(z["objective"])
    assert label_agreement(api.kmeans(y, k, 0), z["labels"]) >= 0.999
    # the device PCG log: max iterations over columns per inner iteration
    assert list(its.max(axis=1)) == list(z["pcg_log"])
    # fp64 in the reference's operation order: far inside the gate
    assert rel_fro_signed(y, z["y"]) <= 1e-9
