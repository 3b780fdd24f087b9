"""C-ABI boundary checks that need no GPU: the library loads, exports exactly
what include/pfe_b200.h declares, refuses to compute without a device (no CPU
fallback), and its host-side boundary helpers reproduce the oracle bitwise."""
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from conftest import random_graph
from paper_1612_06496_b200 import _native as N
from paper_1612_06496_b200 import api

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "pfe_b200.h"


def header_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = set(re.findall(r"\b(pfe_[a-z_0-9]+)\s*\(", text))
    return {n for n in names if not n.endswith("_fn")}


def test_header_declares_and_library_exports_every_symbol():
    lib = N.load()
    declared = header_functions()
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in pfe_b200.h but not exported"
    assert declared == set(N.EXPORTED_SYMBOLS)
    out = subprocess.run(["nm", "-D", "--defined-only", str(N.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (pfe_[a-z_0-9]+)", out))
    assert declared <= exported


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_params_default_mirrors_reference():
    p = N.load().pfe_params_default()
    # solver.hpp:16-25, pcg.hpp:15-19
    assert (p.dim, p.lambda_, p.r, p.soc_max, p.sb_max_stage1, p.sb_max_stage2) == (5, 100.0, 1.0, 10, 5, 100)
    assert (p.conv_tol, p.pcg_rel_tol, p.pcg_max_iter, p.preconditioner) == (1e-4, 1e-6, 1000, 0)


def _have_gpu():
    return N.load().pfe_device_check(0) == 0


@pytest.mark.skipif(_have_gpu(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu(rng):
    assert N.load().pfe_device_check(0) == N.PFE_CONFIG_ERROR
    with pytest.raises(api.ConfigError, match="no CPU fallback|no CUDA device"):
        api.shrink(np.ones(4), 0.5)
    g = random_graph(6, 4, rng)
    with pytest.raises(api.ConfigError):
        api.PfeSolver(g, api.PfeParams(dim=2))


def test_config_errors_precede_device_use(rng):
    g = random_graph(6, 4, rng)
    bad = api.WeightedGraph(g.n, g.ei, g.ej, g.w, np.r_[g.degree[:-1], 0.0])
    with pytest.raises(api.ConfigError, match="nonpositive degree at vertex 5"):
        api.PfeSolver(bad, api.PfeParams(dim=2))
    with pytest.raises(api.ConfigError, match="r must be > 0"):
        api.PfeSolver(g, api.PfeParams(dim=2, r=0.0))
    with pytest.raises(api.ConfigError, match="dim must be >= 1"):
        api.PfeSolver(g, api.PfeParams(dim=0))
    with pytest.raises(api.ConfigError, match="iteration caps"):
        api.PfeSolver(g, api.PfeParams(dim=2, soc_max=0))
    with pytest.raises(api.ConfigError, match="rel_tol"):
        api.PfeSolver(g, api.PfeParams(dim=2, pcg=api.PcgConfig(rel_tol=0.0)))


def test_random_embedding_bitwise_equal_to_oracle(rng):
    g = random_graph(300, 500, rng)
    for d, seed in [(1, 0), (3, 7), (8, 123456789)]:
        a = api.random_embedding(300, d, seed, g.degree)
        b = O.random_embedding(300, d, seed, g.degree)
        assert np.array_equal(a, b)
        gram = a.T @ np.diag(g.degree) @ a
        assert np.abs(gram - np.eye(d)).max() < 1e-8  # test_init.cpp:130-137


def test_d_orthonormalize_dependent_column_rejected():
    a = np.ones((6, 2))
    a[:, 1] = 3.0
    with pytest.raises(api.NumericalError, match="dependent column 1"):
        api.d_orthonormalize(a, np.ones(6))


def test_kmeans_labels_bitwise_equal_to_oracle():
    rng = np.random.Generator(np.random.PCG64(9))
    pts = np.concatenate([rng.normal(0, 0.05, (200, 3)), rng.normal(5, 0.05, (200, 3)),
                          rng.normal(-5, 0.3, (300, 3))])
    for k, seed in [(2, 0), (3, 1), (7, 42)]:
        assert np.array_equal(api.kmeans(pts, k, seed), O.kmeans(pts, k, seed))
    with pytest.raises(api.ConfigError, match="k exceeds point count"):
        api.kmeans(pts[:3], 4, 0)
