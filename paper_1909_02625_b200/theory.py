"""Lemma-1 bookkeeping over device deviation rows.

Host arithmetic on ``DeviationRow`` values (deviation.py), restating the reference's Lemma-1
helpers (/root/reference/pkg/src/stalepipe/theory.py:88-151) in array form: the per-block bound
is L*M times the suffix sum of the snapshot distances over blocks >= k, so one reversed
cumulative sum per row gives every block's bound (and, divided into the measured forward-snapshot
deviation, every block's implied Lipschitz constant). The suffix sums accumulate from the top
block down, the order the reference adds them in, so the numbers agree exactly
(tests/test_oracle_cpu.py::test_theory_port_matches_reference).
"""

from __future__ import annotations

import numpy as np


def _suffix_sums(diffs) -> np.ndarray:
    """s[k] = sum_{j >= k} diffs[j], accumulated from the last block down."""
    d = np.asarray(diffs, dtype=np.float64)
    return np.cumsum(d[::-1])[::-1]


def lemma_bound_rhs(L: float, M: float, diffs) -> list:
    """Per-block Lemma-1 bound L*M * sum_{j >= k} ||x_j(bwd) - x_j(fwd)|| (non-increasing in k)."""
    return list((L * M) * _suffix_sums(diffs))


def estimate_constants(samples) -> tuple:
    """Empirical (L_hat, M_hat) of a run's deviation rows: M_hat is the largest error-gradient
    norm a block received; L_hat the smallest L for which L_hat*M_hat bounds every sampled
    forward-snapshot deviation whose suffix distance is positive."""
    samples = list(samples)
    m_hat = max((max(r.upstream_norms) for r in samples), default=0.0)
    if m_hat <= 0.0:
        return 0.0, m_hat
    l_hat = 0.0
    for r in samples:
        tail = _suffix_sums(r.diffs)
        pos = tail > 0.0
        if pos.any():
            ratio = np.asarray(r.raw_fwd, dtype=np.float64)[pos] / (m_hat * tail[pos])
            l_hat = max(l_hat, float(ratio.max()))
    return l_hat, m_hat


def lemma1_report(samples, L: float, M: float) -> dict:
    """Measured forward-snapshot deviations against the L*M bound; a row holds when every block is
    within its bound (a zero bound demands an exactly zero deviation)."""
    rows = []
    for r in samples:
        bound = lemma_bound_rhs(L, M, r.diffs)
        measured = list(r.raw_fwd)
        rows.append({"batch_index": r.batch_index, "measured": measured, "bound": bound,
                     "holds": bool(np.all(np.asarray(measured) <= np.asarray(bound)))})
    held = sum(row["holds"] for row in rows)
    return {"L": L, "M": M, "samples": len(rows), "holds_fraction": held / len(rows) if rows else 1.0, "rows": rows}
