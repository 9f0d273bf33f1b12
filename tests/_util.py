"""Shared numeric helpers for the GPU parity tests (tolerances from SURVEY.md §8c)."""

import numpy as np

from oracle import oracle as O

REL_L2 = 5e-3
MAX_ABS_FRAC = 2.0 ** -7


def assert_close_bf16(got_u16, ref_u16, what=""):
    """bf16 tensors (uint16 bit patterns) within rel-L2 <= 5e-3 and
    max-abs <= 2^-7 * max|ref| of the oracle."""
    g = O.bf16_to_f32(got_u16).astype(np.float64)
    r = O.bf16_to_f32(ref_u16).astype(np.float64)
    assert np.isfinite(g).all(), f"{what}: non-finite output"
    rel = np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-30)
    mx = np.abs(g - r).max() if g.size else 0.0
    assert rel <= REL_L2, f"{what}: rel-L2 {rel:.3e} > {REL_L2}"
    assert mx <= MAX_ABS_FRAC * max(np.abs(r).max(), 1e-30), f"{what}: max-abs {mx:.3e}"
