"""BASELINE-size parity helpers shared by tests/golden/make_config_fixtures.py
(the CPU oracle side, run in the build container) and the ``-m gpu`` tests
(the CUDA side, run on the B200 box).

A full-size field (config 3: 4.08 M nodes x 5 unknowns) is too large to
commit, so the fixtures hold, per element, two size-independent summaries
of the field plus the full blocks of a seeded element sample:

* ``emax[e]``  = max |x| over the element's nodes and unknowns;
* ``wsum[e]``  = sum_k w_k x_k with fixed pseudo-random weights w in [-1, 1)
  (a hash of element id and node index); ``wabs[e]`` = sum_k |w_k| is
  recomputed from the weights.

If every node of every element agrees to ``tol * scale`` (the pointwise
parity bar), then |d emax| <= tol*scale and |d wsum| <= tol*scale*wabs: both
are necessary conditions of the bar, checked for EVERY element, and a wrong
node anywhere moves its element's weighted sum.  The sample is compared
pointwise.

Both sides compute the summaries from the oracle's bucket-block layout
(B, nv, n1+1, n2+1, n3+1); the GPU field is converted with
``NodalField.to_oracle_blocks``.
"""

from __future__ import annotations

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SAMPLE = 64


def weights(elem_ids, k):
    """Fixed weights in [-1, 1) for k values of each element in elem_ids."""
    x = np.asarray(elem_ids, dtype=np.float64)[:, None] * 12.9898 + np.arange(k)[None, :] * 78.233
    s = np.sin(x) * 43758.5453
    return 2.0 * (s - np.floor(s)) - 1.0


def element_stats(orders, blocks):
    """(emax, wsum, wabs) per element id from oracle-layout bucket blocks.

    ``orders``: any object with ``num_elements``, ``group_elements``."""
    nel = orders.num_elements
    emax, wsum, wabs = np.zeros(nel), np.zeros(nel), np.zeros(nel)
    for ids, blk in zip(orders.group_elements, blocks):
        flat = np.asarray(blk).reshape(len(ids), -1)
        w = weights(ids, flat.shape[1])
        emax[ids] = np.abs(flat).max(axis=1)
        wsum[ids] = (w * flat).sum(axis=1)
        wabs[ids] = np.abs(w).sum(axis=1)
    return emax, wsum, wabs


def sample_elements(nel, seed=0, k=SAMPLE):
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(nel, size=min(k, nel), replace=False))


def element_block(orders, blocks, e):
    g, r = (int(x) for x in orders.element_slot[e])
    return np.asarray(blocks[g][r])


def sample_values(orders, blocks, elems):
    return np.concatenate([element_block(orders, blocks, int(e)).ravel() for e in elems])


def field_summary(prefix, orders, blocks, sample):
    """Fixture entries for one field."""
    emax, wsum, _ = element_stats(orders, blocks)
    return {f"{prefix}_emax": emax, f"{prefix}_wsum": wsum,
            f"{prefix}_sample": sample_values(orders, blocks, sample)}


def compare_field(fx, prefix, orders, blocks, scale, tol=1e-12):
    """Assert the GPU field (oracle-layout blocks) matches the fixture; returns
    the measured worst errors relative to ``scale``."""
    emax, wsum, wabs = element_stats(orders, blocks)
    e_max = float(np.abs(emax - fx[f"{prefix}_emax"]).max()) / scale
    e_sum = float((np.abs(wsum - fx[f"{prefix}_wsum"]) / wabs).max()) / scale
    samp = sample_values(orders, blocks, fx["sample"])
    e_pt = float(np.abs(samp - fx[f"{prefix}_sample"]).max()) / scale
    assert e_max <= tol, f"{prefix}: element max|x| off by {e_max:.3e} (relative)"
    assert e_sum <= tol, f"{prefix}: element weighted sum off by {e_sum:.3e} (relative)"
    assert e_pt <= tol, f"{prefix}: sampled nodes off by {e_pt:.3e} (relative)"
    return {"emax": e_max, "wsum": e_sum, "sample": e_pt}


def tau_dense(tmap, nel, nmax=8):
    """TauMap -> (nel, 3, nmax) array, NaN where no entry."""
    out = np.full((nel, 3, nmax), np.nan)
    for e in range(nel):
        for d in range(3):
            for n, v in tmap.tau[e][d].items():
                if n < nmax:
                    out[e, d, n] = v
    return out


def load(name):
    return dict(np.load(os.path.join(GOLDEN, f"oracle_{name}.npz"), allow_pickle=False))


def have(name):
    return os.path.exists(os.path.join(GOLDEN, f"oracle_{name}.npz"))
