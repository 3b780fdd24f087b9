"""Small repro of the tiled persistent kernel (TMA staging) for debugging."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from conftest import *  # noqa
from test_gpu_solver import small_image, jacobi
from paper_1612_06496_b200 import api
radius = int(sys.argv[1]) if len(sys.argv) > 1 else 1
d = int(sys.argv[2]) if len(sys.argv) > 2 else 4
g = small_image(48, 70, seed=5, radius=radius, sigma_xy=2.0 if radius == 2 else None)
prm = jacobi(d, soc=1, sb=2)
y0 = api.random_embedding(g.n, d, 4, g.degree)
s = api.PfeSolver(g, prm, warn=False, persistent="tiled")
st = s.make_state(y0)
s.run_soc(st, 1, 2)
print("ok", s.report())
