"""Times GPU k-means (pfe_kmeans_device) on a C4-sized embedding (n x d, k)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np

    from paper_1612_06496_b200 import api

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16_777_216
    d = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    k = int(sys.argv[3]) if len(sys.argv) > 3 else 256
    it = int(sys.argv[4]) if len(sys.argv) > 4 else 20
    rng = np.random.Generator(np.random.PCG64(0))
    centres = rng.uniform(-1, 1, size=(k, d))
    pts = centres[rng.integers(0, k, size=n)] + rng.normal(0, 0.05, size=(n, d))
    api.kmeans(pts[:1000], 4, 0, device=0)
    t0 = time.perf_counter()
    lab = api.kmeans(pts, k, 0, max_iter=it, device=0)
    dt = time.perf_counter() - t0
    print(f"device kmeans n={n} d={d} k={k} max_iter={it}: {dt:.2f} s, {len(np.unique(lab))} clusters used")
    if n <= 2_000_000:
        t0 = time.perf_counter()
        host = api.kmeans(pts, k, 0, max_iter=it)
        print(f"host kmeans: {time.perf_counter() - t0:.2f} s, equal labels {np.mean(host == lab):.6f}")


if __name__ == "__main__":
    main()
