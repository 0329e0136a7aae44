"""Fit the reference's linear stage cost model to measured B200 stage times.

The reference simulator charges every micro-batch
    stage_ms = c0 + c_tok * total_tokens + c_ctx * decode_context_tokens / 1024
(`pkg/src/tokensim/engine.py:96-100`, coefficients `StageCostModel`, `engine.py:45-57`).
Given (total_tokens, decode_context_tokens, measured device ms) per micro-batch
from a GPU run, a non-negative least-squares fit returns the coefficients that
make the virtual-clock engine (here or in the reference) predict B200 timing,
so simulated and measured TTFT/TPOT/bubble become comparable.
"""

from __future__ import annotations

import numpy as np

from .engine import StageCostModel


def fit_stage_cost(total_tokens, decode_context_tokens, stage_ms, n_stages: int = 1) -> tuple[StageCostModel, dict]:
    """NNLS fit of (c0, c_tok, c_ctx) per stage; returns the model and fit diagnostics.

    `stage_ms` is the measured time of the whole micro-batch on the device holding
    all `n_stages` stages; each stage is charged 1/n_stages of it (uniform stages,
    D-E1 `SPEC.md:388`).
    """
    tok = np.asarray(total_tokens, dtype=np.float64)
    ctx = np.asarray(decode_context_tokens, dtype=np.float64) / 1024.0
    y = np.asarray(stage_ms, dtype=np.float64) / n_stages
    if tok.size < 3:
        raise ValueError("need at least 3 micro-batches to fit 3 coefficients")
    X = np.stack([np.ones_like(tok), tok, ctx], axis=1)
    coef = _nnls(X, y)
    pred = X @ coef
    rel = np.abs(pred - y) / np.maximum(y, 1e-9)
    model = StageCostModel(c0=float(coef[0]), c_tok=float(coef[1]), c_ctx=float(coef[2]))
    return model, {"n": int(tok.size), "mean_abs_rel_err": float(rel.mean()), "max_abs_rel_err": float(rel.max()),
                   "r2": float(1.0 - ((pred - y) ** 2).sum() / max(((y - y.mean()) ** 2).sum(), 1e-12))}


def _nnls(X: np.ndarray, y: np.ndarray, iters: int = 200) -> np.ndarray:
    """Small active-set NNLS (3 columns): least squares with coefficients clipped to >= 0."""
    active = list(range(X.shape[1]))
    for _ in range(iters):
        coef = np.zeros(X.shape[1])
        sol, *_ = np.linalg.lstsq(X[:, active], y, rcond=None)
        coef[active] = sol
        neg = [a for a, c in zip(active, sol) if c < 0]
        if not neg:
            return coef
        active = [a for a in active if a not in neg]
        if not active:
            return np.zeros(X.shape[1])
    return np.clip(coef, 0.0, None)
