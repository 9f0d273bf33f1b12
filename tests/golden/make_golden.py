"""Regenerates the golden fixtures under tests/golden/ from the oracle.

The reference ships no golden vectors for this path, so these
are self-generated regression vectors that pin the oracle's (and therefore the
GPU path's) bit-exact outputs; run this script only when the precision
contract in DESIGN.md §3 changes on purpose.

  python tests/golden/make_golden.py
"""

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402

CASES = {
    "tiny": (64, 512, 1536, 8, 2),       # config 1 shape
    "dbrx_router": (48, 6144, 128, 16, 4),
    "deepseek_router": (24, 7168, 128, 256, 8),
}


def main():
    for name, (T, H, Hp, E, K) in CASES.items():
        wts = O.synth_weights(H, Hp, E, seed=0, experts=None if name == "tiny" else [])
        x = O.synth_tokens(T, H, seed=1)
        idx, w, lg = O.router(x, wts.wg, K, want_logits=True)
        cnt, slot = O.place(idx, E)
        # inputs are regenerated from their seeds by the test; their SHA-256 is
        # pinned here so generator drift is caught, not silently absorbed
        out = dict(x_sha=np.frombuffer(hashlib.sha256(x.tobytes()).digest(), np.uint8),
                   wg_sha=np.frombuffer(hashlib.sha256(wts.wg.tobytes()).digest(), np.uint8),
                   shape=np.array([T, H, Hp, E, K]), idx=idx, w=w, logits=lg, cnt=cnt, slot=slot)
        if name == "tiny":
            res = O.moe_layer([x], wts, K, n_e=1, resid=True)
            out.update(y=res.y[0], out=res.out[0])
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(name, "written")


if __name__ == "__main__":
    main()
