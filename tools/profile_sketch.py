"""ncu driver: one C2 ritzit and one REVD sketch (device-resident Omega)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2101_07249_b200 as W  # noqa: E402
from paper_2101_07249_b200 import configs  # noqa: E402

wl = configs.config2()
op = wl.hessian(0)
Om = W.gaussian_matrix(op.dim(), wl.m, 1)
for method in sys.argv[1:] or ["ritzit"]:
    W.sketch_eigenpairs(op, W.SketchConfig(wl.k, wl.m - wl.k, 1, method), Om)
    print(method, W.last_sketch_timing())
