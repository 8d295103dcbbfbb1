"""Oracle: QoE model fitting (§4.1) — TEST INFRASTRUCTURE ONLY.

  PAPER.md:317-323  fit D_0..D_4 by "a least-squares regression of Q against F_k":
                    (D_0..D_4) = argmin_D sum_j (Q^(j) - sum_k D_k F_k^(j))^2
  PAPER.md:325      validation: relative prediction error on a held-out split (Fig. 13)

Reading Z38: a column mask selects which features enter the fit (decode-only profiles
have no prefill, so F_2 = sum I and F_3 = sum I^2 carry no signal there); masked-out
coefficients are 0.  The step is a library primitive (numpy.linalg.lstsq), as allowed for
an oracle step; rank < number of selected columns is an error.
"""
from __future__ import annotations

import numpy as np


class TooFewSamples(ValueError):
    pass


class RankDeficient(ValueError):
    pass


def fit_params(F, Q, mask=(1, 1, 1, 1, 1)):
    F = np.asarray(F, dtype=np.float64).reshape(-1, 5)
    Q = np.asarray(Q, dtype=np.float64).reshape(-1)
    cols = [k for k in range(5) if mask[k]]
    if F.shape[0] < len(cols) or F.shape[0] < 1:
        raise TooFewSamples(f"{F.shape[0]} samples for {len(cols)} coefficients")
    A = F[:, cols]
    if np.linalg.matrix_rank(A / np.maximum(np.abs(A).max(axis=0), 1e-300)) < len(cols):
        raise RankDeficient("feature matrix is rank deficient")
    sol, *_ = np.linalg.lstsq(A, Q, rcond=None)
    D = np.zeros(5)
    D[cols] = sol
    return D


def prediction_error(D, F, Q):
    """Per-sample relative error (predicted - actual) / actual and the mean absolute value."""
    F = np.asarray(F, dtype=np.float64).reshape(-1, 5)
    Q = np.asarray(Q, dtype=np.float64)
    pred = F @ np.asarray(D, dtype=np.float64)
    rel = (pred - Q) / Q
    return rel, float(np.mean(np.abs(rel)))
