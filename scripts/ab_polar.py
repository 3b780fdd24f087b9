"""Bitwise A/B of the projection (TSQR + Jacobi SVD + apply) between the
library in use (PFE_LIB_VARIANT selects a variant) and saved outputs."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_1612_06496_b200 import api
out = Path(sys.argv[1])
mode = sys.argv[2]  # save | check
rng = np.random.Generator(np.random.PCG64(5))
cases = [(300, 3), (1000, 4), (5000, 8), (70000, 8), (250000, 16), (40000, 5), (2000, 12), (333, 1), (100000, 2)]
res = {}
for n, d in cases:
    a = rng.normal(size=(n, d)) * rng.uniform(0.1, 3.0, size=(1, d))
    a[:, -1] += 0.5 * a[:, 0]
    if d > 2:
        a[::7, 1] = 0.0
        a[:n // 3, 2] = -0.0
    res[f"{n}x{d}"] = api.project_orthogonal(a)
if mode == "save":
    np.savez(out, **res)
else:
    ref = np.load(out)
    for k, v in res.items():
        same = np.array_equal(v, ref[k])
        print(k, "bitwise equal" if same else f"DIFFERENT max {np.abs(v - ref[k]).max():.3e}")
        assert same
    print("all projections bit-identical")
