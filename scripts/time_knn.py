"""Times the GPU k-NN graph build of a config (C5 by default)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np

    from paper_1612_06496_b200 import api

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    rng = np.random.Generator(np.random.PCG64(0))
    means = rng.uniform(-10.0, 10.0, size=(32, 16))
    stds = rng.uniform(0.5, 1.5, size=32)
    wts = rng.exponential(1.0, size=32)
    wts /= wts.sum()
    comp = rng.choice(32, size=n, p=wts)
    pts = means[comp] + rng.normal(size=(n, 16)) * stds[comp, None]
    api.knn_graph_gpu(pts[:1000], 16)  # context
    t0 = time.perf_counter()
    g = api.knn_graph_gpu(pts, 16)
    dt = time.perf_counter() - t0
    print(f"n={n} m={g.m} m/n={g.m / n:.2f} sigma={g.sigma:.6f} build {dt:.2f} s")


if __name__ == "__main__":
    main()
