"""Full-size goldens (tests/golden/full_<cfg>.npz, made by
tests/golden/make_full_golden.py with the column-parallel oracle): CPU checks
that pin them to this repo's input generators and to the oracle's own
bookkeeping.  The GPU comparison is tests/test_gpu_full_parity.py.
"""
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from golden.make_full_golden import SAMPLE_ROWS, array_sha, block_sums, evidence, graph_sha
from paper_1612_06496_b200.inputs import make_config

GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_full_golden_is_consistent(name):
    z = np.load(GOLDEN / f"full_{name}.npz")
    n, d = int(z["n"]), int(z["d"])
    assert len(z["pcg_log"]) == int(z["soc_max"]) * int(z["sb_max"])
    assert z["labels"].shape == (n,) and int(z["labels"].max()) < int(z["k"])
    assert z["y_rows"].shape == (len(z["rows"]), d) and len(z["rows"]) >= SAMPLE_ROWS
    assert np.array_equal(z["rows"], np.arange(0, n, int(z["stride"])))
    assert z["block_sums"].shape == ((n + 4095) // 4096, d)
    # the Gram diagonal is the squared column norms
    assert np.allclose(np.diag(z["gram"]), z["col_norms"] ** 2, rtol=1e-12)
    assert abs(np.sqrt(np.sum(z["col_norms"] ** 2)) - float(z["fro"])) <= 1e-12 * float(z["fro"])
    assert 0.0 < float(z["objective"]) < float(z["objective0"])


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_full_golden_inputs_match_generators(name):
    """The pixel-grid graphs and Y0 the goldens were made from are what
    inputs.make_config and random_embedding produce today (C5's graph is built
    on the GPU; its hash is checked by the GPU test)."""
    z = np.load(GOLDEN / f"full_{name}.npz")
    cfg = make_config(name)
    g = cfg.graph
    assert graph_sha(g) == str(z["graph_sha"])
    y0 = O.random_embedding(g.n, cfg.params.dim, cfg.y0_seed, g.degree)
    assert array_sha(np.asfortranarray(y0)) == str(z["y0_sha"])


def test_evidence_is_sign_and_row_faithful():
    """The summaries the GPU test compares see every row (block sums) and
    flip with a column sign like Y does."""
    rng = np.random.Generator(np.random.PCG64(0))
    y = rng.normal(size=(10000, 3))
    e = evidence(y)
    y2 = y.copy()
    y2[9999, 1] += 1e-3
    assert not np.array_equal(block_sums(y2), e["block_sums"])
    s = np.array([1.0, -1.0, 1.0])
    assert np.allclose(block_sums(y * s), e["block_sums"] * s)


def test_oracle_session_follows_the_soc_schedule():
    """bench.py's CPU legs step a resident oracle solve one inner iteration at a
    time; the trajectory equals the one-call soc bit for bit."""
    cfg = make_config("c2", scale=(30, 40))
    g, prm = cfg.graph, cfg.params
    prm.soc_max, prm.sb_max_stage1 = 3, 4
    y0 = O.random_embedding(g.n, prm.dim, 0, g.degree)
    full = O.solve_timed(g, prm, y0)
    s = O.Session(g, prm, y0)
    ks = np.concatenate([s.step(1)[2] for _ in range(prm.soc_max * prm.sb_max_stage1)])
    s.close()
    assert np.array_equal(ks, full["pcg_log"])
    assert full["t_inner"] > 0.0 and full["t_setup"] > 0.0
