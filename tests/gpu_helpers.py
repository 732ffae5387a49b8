"""Helpers shared by the GPU parity tests (no test functions here)."""
import numpy as np


def check_trace_panels(tr, panels, jpvt_o, first=0, last=None, tol=1e-12, k=None):
    """Per recorded panel: the pivots exactly; R-hat after the sample QRCP
     and the updated sample B_next (Eq. (4)) in the
    Frobenius norm to tol * ||B_0||_F, B_0 = Omega A the initial sample
    (= ||R-hat of panel 0||_F: an orthogonal transform).  Every later sample
    is an orthogonal / triangular transform of Omega times a trailing part of
    A, and the rounding it inherits from the trailing updates (which cancel
    down to the noise level on low-rank inputs) is relative
    to the data it came from, i.e. to ||Omega A||, not to its own size."""
    scale = np.linalg.norm(panels[0][2])
    for t, (i, bb, Rh_o, Bn_o) in enumerate(panels):
        if t < first or (last is not None and t >= last):
            continue
        piv, Rh_g, Bn_g = tr.panel(t, bb, i)
        assert np.array_equal(piv, jpvt_o[i:i + bb]), f"panel {t}: pivots"
        assert np.linalg.norm(Rh_g - Rh_o) <= tol * scale, f"panel {t}: R-hat"
        gpu_updates = k is None or i + bb < k  # no sample update after the last panel (R-G9)
        if Bn_o is not None and Bn_o.shape[1] > 0 and gpu_updates:
            assert np.linalg.norm(Bn_g - Bn_o) <= tol * scale, f"panel {t}: B_next"
