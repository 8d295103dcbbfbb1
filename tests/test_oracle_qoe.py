"""Pins for the QoE-fit oracle (oracle/qoe.py): SPEC.md fit_params / prediction_error examples
 and OLS properties."""
import numpy as np
import pytest

from oracle import qoe as oq


def _features(rng, n):
    rows = []
    for _ in range(n):
        b = int(rng.integers(1, 64))
        I = rng.integers(1, 4000, size=b)
        L = I + rng.integers(1, 2000, size=b)
        rows.append([1, b, I.sum(), (I * I).sum(), L.sum()])
    return np.array(rows, dtype=np.float64)


def test_noiseless_recovery():
    """samples generated noiselessly from known D* -> D* within 1e-6 relative."""
    rng = np.random.default_rng(0)
    F = _features(rng, 40)
    Dstar = np.array([2e-2, 3e-4, 1e-6, 2e-11, 5e-7])
    D = oq.fit_params(F, F @ Dstar)
    assert np.max(np.abs(D - Dstar) / np.abs(Dstar)) < 1e-6


def test_constant_q_and_errors():
    rng = np.random.default_rng(1)
    F = _features(rng, 12)
    D = oq.fit_params(F, np.full(12, 0.7))               # constant Q -> (c, 0, 0, 0, 0)
    assert abs(D[0] - 0.7) < 1e-9 and np.max(np.abs(D[1:] * F[:, 1:].max(axis=0))) < 1e-8
    with pytest.raises(oq.TooFewSamples):
        oq.fit_params(F[:3], np.ones(3))
    G = F.copy()
    G[:, 4] = 2 * G[:, 2]                               # collinear columns -> rank deficient
    with pytest.raises(oq.RankDeficient):
        oq.fit_params(G, np.ones(12))
    D3 = oq.fit_params(G, G @ np.array([1.0, 2.0, 0.0, 0.0, 3.0]), mask=(1, 1, 0, 0, 1))
    assert D3[2] == 0 and D3[3] == 0 and abs(D3[4] - 3.0) < 1e-6


def test_residual_orthogonal_and_prediction_error():
    rng = np.random.default_rng(2)
    F = _features(rng, 30)
    Q = F @ np.array([1e-2, 1e-4, 1e-7, 0.0, 1e-6]) * rng.uniform(0.9, 1.1, size=30)
    D = oq.fit_params(F, Q)
    r = Q - F @ D
    for k in range(5):                                   # S:105 OLS residual orthogonality
        assert abs(np.dot(r, F[:, k])) < 1e-6 * np.linalg.norm(r) * np.linalg.norm(F[:, k]) + 1e-12
    rel, mean = oq.prediction_error(D, F, F @ D)
    assert mean == 0.0                                   # S:95 noiseless -> all errors 0
    rel2, _ = oq.prediction_error(D, F, 2 * (F @ D))     # S:96 doubled actual -> -0.5
    assert np.allclose(rel2, -0.5)
