"""Times the GPU GMM initial embedding (pfe_gmm_init_device) on a config's
image (C2: 481x321, C4: 4096x4096) with k = d, and the CPU oracle on C2.

usage: python scripts/time_gmm.py [config]
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    import numpy as np

    from paper_1612_06496_b200 import api
    from paper_1612_06496_b200.inputs import grid_graph, voronoi_image

    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    h, w, regions, k = {"c2": (321, 481, 8, 4), "c4": (4096, 4096, 256, 8)}[name]
    rng = np.random.Generator(np.random.PCG64(0))
    img, _ = voronoi_image(h, w, regions, 0.05, rng)
    f = img.reshape(-1, 3)
    deg = grid_graph(img, 0.1, 1).degree
    api.gmm_init_embedding(f[:4096], k, 0, deg[:4096])  # context
    t0 = time.perf_counter()
    y = api.gmm_init_embedding(f, k, 0, deg)
    dt = time.perf_counter() - t0
    print(f"{name}: GPU gmm init n={f.shape[0]} k={k}: {dt:.3f} s")
    if name == "c2":
        import oracle as O

        t0 = time.perf_counter()
        exp = O.gmm_init_embedding(f, k, 0, deg)
        dc = time.perf_counter() - t0
        print(f"{name}: CPU oracle gmm init (1 core): {dc:.3f} s; rel diff {np.linalg.norm(y - exp) / np.linalg.norm(exp):.2e}")


if __name__ == "__main__":
    main()
