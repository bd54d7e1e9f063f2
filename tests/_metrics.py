"""Parity metric of SURVEY.md §8(c) Q11 (also DESIGN.md §3): max |x_hat - x| / max(|x|, floor)."""
import numpy as np


def max_rel_err(x_hat, x, floor):
    x_hat = np.asarray(x_hat, np.float64)
    x = np.asarray(x, np.float64)
    assert x_hat.shape == x.shape, (x_hat.shape, x.shape)
    if x.size == 0:
        return 0.0
    den = np.maximum(np.abs(x), floor)
    return float(np.max(np.abs(x_hat - x) / den))


def flow_floor(problem):
    """F floor: 1e-30 * m_tot (Q11)."""
    mass = problem.mass if problem.is_point else problem.mu0.sum(axis=1)
    return 1e-30 * float(np.sum(mass))


W_FLOOR = 1e-30
