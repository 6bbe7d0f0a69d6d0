"""Random initial configurations (the init / fill kernel of SURVEY §2.3 N-K3; reading R32).

TEST INFRASTRUCTURE (see oracle/__init__.py).

The paper starts its runs from given coverages (an empty lattice; Bernoulli coverages for
the phase diagrams) and fixes no generator.  R32: site x = (x, y) of replica r takes state
s = #{j < S-1 : u >= T_j} with u = word 0 of Philox4x32-10(ctr = (x, y, r, TAG_INIT << 28),
key = seed) and thresholds T_j = floor(2^32 (p_0 + ... + p_j)) (2^32 when the partial sum reaches 1),
so P(s) = p_s up to 2^-32 and the state of a site depends only on (seed, global site) -- not on
the rank split or the launch shape.  Written out below site by site.
"""
import math

import numpy as np

from . import philox4x32_10

TAG_INIT = 2


def thresholds(probs):
    """T_j for j = 0 .. S-2 (R32)."""
    probs = [float(p) for p in probs]
    if any(not (p >= 0.0) for p in probs):
        raise ValueError("probabilities must be >= 0")
    out, c = [], 0.0
    for p in probs[:-1]:
        c = c + p
        if c > 1.0 + 1e-12:
            raise ValueError("partial sums of the probabilities exceed 1")
        out.append(1 << 32 if c >= 1.0 else int(math.floor(c * 4294967296.0)))
    return out


def init_random(R, H, W, probs, seed, row_offset=0, rep_offset=0):
    """[R][H][W] uint8 states of the local slab (rows row_offset.., replicas rep_offset..)."""
    T = thresholds(probs)
    key = (seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    lat = np.zeros((R, H, W), dtype=np.uint8)
    for r in range(R):
        for y in range(H):
            for x in range(W):
                u = philox4x32_10((x, y + row_offset, r + rep_offset, TAG_INIT << 28), key)[0]
                lat[r, y, x] = sum(1 for t in T if u >= t)
    return lat
