"""Exact Kalman filter for the linear-Gaussian HMMs (test oracle for the filter mean).

TEST INFRASTRUCTURE ONLY.  PAPER.md:1253 ("admits exact numerical calculation by
Kalman filter recursions"); dense fp64 with the Joseph-form covariance update
(SPEC.md:112); posterior after the update at every n, including n = 0
(SPEC.md:89, 120).

Model: X_0 ~ N(m0, P0), X_n = A X_{n-1} + N(0, Q), Y_n = H X_n + N(0, R).
"""
from __future__ import annotations

import numpy as np


def kalman_filter(A, Q, H, R, m0, P0, ys):
    """Returns (means[T, d], covs[T, d, d]) of p(x_n | y_{0:n})."""
    A = np.asarray(A, np.float64)
    Q = np.asarray(Q, np.float64)
    H = np.asarray(H, np.float64)
    R = np.asarray(R, np.float64)
    m = np.asarray(m0, np.float64).copy()
    P = np.asarray(P0, np.float64).copy()
    d = m.shape[0]
    ys = np.asarray(ys, np.float64)
    if not np.all(np.isfinite(ys)):
        raise ValueError("non-finite observation")
    means = np.zeros((len(ys), d))
    covs = np.zeros((len(ys), d, d))
    I = np.eye(d)
    for n, y in enumerate(ys):
        if n > 0:
            m = A @ m
            P = A @ P @ A.T + Q
        Sm = H @ P @ H.T + R
        K = P @ H.T @ np.linalg.inv(Sm)
        m = m + K @ (y - H @ m)
        IKH = I - K @ H
        P = IKH @ P @ IKH.T + K @ R @ K.T
        P = 0.5 * (P + P.T)
        means[n] = m
        covs[n] = P
    return means, covs


def kalman_scalar(a, q, r, m0, p0, ys):
    """Scalar recursion (d = 1, H = 1) written out by hand; cross-check of the dense one."""
    m, p = float(m0), float(p0)
    out_m, out_p = [], []
    for n, y in enumerate(ys):
        if n > 0:
            m = a * m
            p = a * a * p + q
        k = p / (p + r)
        m = m + k * (float(y) - m)
        p = (1.0 - k) * p
        out_m.append(m)
        out_p.append(p)
    return np.array(out_m), np.array(out_p)
