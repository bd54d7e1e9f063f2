"""ORACLE PINS (test infrastructure only): representation twins of the log-domain oracle.

Twin A: Algorithm 2 (alg:multi_commodity P:1085-1107) in the LINEAR domain with a configurable
scalar dtype (np.longdouble = x87 80-bit: 64-bit significand, range ~e^+-11356), node form:

    alpha_0 = U0^T,  alpha_{t+1} = (K_t ⊙ W_t)^T alpha_t           (eq:psi_hat)
    beta_T  = UT^T,  beta_t      = (K_t ⊙ W_t)   beta_{t+1}         (eq:psi,     P:1038-1043)
    U0 = mu0 ./ beta_0^T;  W_t = min(d ./ (K_t ⊙ (alpha_t beta_{t+1}^T)) , 1);
    UT = muT ./ alpha_T^T

Twin B: the same recursion with mpmath multiprecision scalars (pure-Python loops; micro only).
Neither twin shares code with oracle/sweep.py.
"""
from __future__ import annotations

import numpy as np


def _spmv_into(out_rows: np.ndarray, src_rows: np.ndarray, weight: np.ndarray, x: np.ndarray, n: int, dtype):
    """y[v, :] = sum_{a : out_rows[a] = v} weight[a] * x[src_rows[a], :]  (plain accumulation)."""
    y = np.zeros((n, x.shape[1]), dtype=dtype)
    np.add.at(y, out_rows, weight[:, None] * x[src_rows])
    return y


class LinearTwin:
    def __init__(self, problem, dtype=np.longdouble):
        p = problem
        self.p, self.dt = p, dtype
        T, A = p.T, p.A
        cost = np.broadcast_to(p.cost, (T, A)) if p.cost.ndim == 1 else p.cost
        self.K = np.exp(-np.asarray(cost, dtype) / dtype(p.eps))
        self.cap = np.broadcast_to(p.cap, (T, A)).astype(dtype) if p.cap.ndim == 1 else p.cap.astype(dtype)
        self.W = np.ones((T, A), dtype)
        self.mu0 = p.mu0.astype(dtype)
        self.muT = p.muT.astype(dtype)
        self.UT = (self.muT > 0).astype(dtype)
        self.U0 = np.zeros_like(self.mu0)
        self.alpha = np.zeros((T + 1, p.N, p.L), dtype)
        self.beta = np.zeros((T + 1, p.N, p.L), dtype)
        self._backward()

    def _backward(self):
        p = self.p
        self.beta[p.T] = self.UT.T
        for t in range(p.T - 1, -1, -1):
            self.beta[t] = _spmv_into(p.tail, p.head, self.K[t] * self.W[t], self.beta[t + 1], p.N, self.dt)

    @staticmethod
    def _div(num, den):
        out = np.zeros_like(num)
        pos = den > 0
        out[pos] = num[pos] / den[pos]
        if ((~pos) & (num > 0)).any():
            raise RuntimeError("infeasible")
        return out

    def sweep(self):
        p = self.p
        self.U0 = self._div(self.mu0, self.beta[0].T)
        self.alpha[0] = self.U0.T
        for t in range(p.T):
            s = (self.alpha[t][p.tail] * self.beta[t + 1][p.head]).sum(axis=1) * self.K[t]
            cap = self.cap[t]
            w = np.ones(p.A, self.dt)
            fin = np.isfinite(cap)
            pos = fin & (s > 0)
            w[pos] = np.minimum(cap[pos] / s[pos], 1)
            w[fin & (cap == 0)] = 0
            self.W[t] = w
            self.alpha[t + 1] = _spmv_into(p.head, p.tail, self.K[t] * self.W[t], self.alpha[t], p.N, self.dt)
        self.UT = self._div(self.muT, self.alpha[p.T].T)
        self._backward()

    def flows(self) -> np.ndarray:
        p = self.p
        return np.stack([(self.alpha[t][p.tail] * self.beta[t + 1][p.head]).sum(axis=1) * self.K[t] * self.W[t]
                         for t in range(p.T)])


class MpTwin:
    """Twin B: same recursion, mpmath scalars, explicit loops (micro instances only)."""

    def __init__(self, problem, dps: int = 40):
        import mpmath
        self.mp = mpmath.mp.clone() if hasattr(mpmath.mp, "clone") else mpmath.mp
        self.mp.dps = dps
        mp = self.mp
        p = problem
        self.p = p
        self.K = [[mp.exp(-mp.mpf(float(p.cost_t(t)[a])) / mp.mpf(p.eps)) for a in range(p.A)] for t in range(p.T)]
        self.cap = [[float(p.cap_t(t)[a]) for a in range(p.A)] for t in range(p.T)]
        self.W = [[mp.mpf(1) for _ in range(p.A)] for _ in range(p.T)]
        self.mu0 = [[mp.mpf(float(x)) for x in row] for row in p.mu0]
        self.muT = [[mp.mpf(float(x)) for x in row] for row in p.muT]
        self.UT = [[mp.mpf(1) if x > 0 else mp.mpf(0) for x in row] for row in self.muT]
        self.U0 = None
        self.beta = None
        self.alpha = None
        self._backward()

    def _backward(self):
        p, mp = self.p, self.mp
        beta = [None] * (p.T + 1)
        beta[p.T] = [[self.UT[l][v] for l in range(p.L)] for v in range(p.N)]
        for t in range(p.T - 1, -1, -1):
            nb = [[mp.mpf(0) for _ in range(p.L)] for _ in range(p.N)]
            for a in range(p.A):
                i, j = int(p.tail[a]), int(p.head[a])
                kw = self.K[t][a] * self.W[t][a]
                for l in range(p.L):
                    nb[i][l] += kw * beta[t + 1][j][l]
            beta[t] = nb
        self.beta = beta

    def sweep(self):
        p, mp = self.p, self.mp
        U0 = [[(self.mu0[l][v] / self.beta[0][v][l]) if self.mu0[l][v] > 0 else mp.mpf(0) for v in range(p.N)]
              for l in range(p.L)]
        self.U0 = U0
        alpha = [None] * (p.T + 1)
        alpha[0] = [[U0[l][v] for l in range(p.L)] for v in range(p.N)]
        for t in range(p.T):
            for a in range(p.A):
                cap = self.cap[t][a]
                if cap == float("inf"):
                    self.W[t][a] = mp.mpf(1)
                    continue
                if cap == 0:
                    self.W[t][a] = mp.mpf(0)
                    continue
                i, j = int(p.tail[a]), int(p.head[a])
                s = mp.fsum(alpha[t][i][l] * self.beta[t + 1][j][l] for l in range(p.L)) * self.K[t][a]
                self.W[t][a] = mp.mpf(1) if s == 0 else min(mp.mpf(cap) / s, mp.mpf(1))
            na = [[mp.mpf(0) for _ in range(p.L)] for _ in range(p.N)]
            for a in range(p.A):
                i, j = int(p.tail[a]), int(p.head[a])
                kw = self.K[t][a] * self.W[t][a]
                for l in range(p.L):
                    na[j][l] += alpha[t][i][l] * kw
            alpha[t + 1] = na
        self.alpha = alpha
        self.UT = [[(self.muT[l][v] / alpha[p.T][v][l]) if self.muT[l][v] > 0 else mp.mpf(0) for v in range(p.N)]
                   for l in range(p.L)]
        self._backward()

    def flows(self):
        p = self.p
        out = np.zeros((p.T, p.A))
        for t in range(p.T):
            for a in range(p.A):
                i, j = int(p.tail[a]), int(p.head[a])
                s = sum(self.alpha[t][i][l] * self.beta[t + 1][j][l] for l in range(p.L))
                out[t, a] = float(s * self.K[t][a] * self.W[t][a])
        return out
