"""Bitwise check of the single-column Fourier-space apply across window-kernel CTA widths:
run once per WC4DVAR_SPECTRAL_W1T value (320 = the wide CTA) and compare the printed digests."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2101_07249_b200 as W  # noqa: E402
from paper_2101_07249_b200 import configs  # noqa: E402

for name, mk in (("C4", lambda: configs.config4(16)),):
    op = mk().hessian(0)
    v = np.asarray(W.gaussian_matrix(op.dim(), 1, 5))[:, 0].copy()
    y = op.apply(v)
    print(name, hashlib.sha256(np.ascontiguousarray(y).tobytes()).hexdigest()[:16], float(np.abs(y).max()))
