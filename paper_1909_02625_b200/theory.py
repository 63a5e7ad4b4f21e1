"""Lemma-1 bookkeeping over device deviation rows.

Host arithmetic on ``DeviationRow`` values, restating
/root/reference/pkg/src/stalepipe/theory.py:88-151 so the rows the B200 engine
produces (deviation.py) feed the same report the reference prints.
"""

from __future__ import annotations


def lemma_bound_rhs(L: float, M: float, diffs) -> list:
    """Right-hand side of Lemma 1 per block: L*M * sum_{j >= k} ||x_j(bwd) - x_j(fwd)||
    (theory.py:88-99)."""
    k_total = len(diffs)
    tail = 0.0
    rhs = [0.0] * k_total
    for k in range(k_total - 1, -1, -1):
        tail += diffs[k]
        rhs[k] = L * M * tail
    return rhs


def estimate_constants(samples) -> tuple:
    """Empirical (L_hat, M_hat): M_hat = largest error-gradient norm any block received;
    L_hat = smallest L making the bound hold at every sampled step with a positive
    snapshot distance (theory.py:102-120)."""
    m_hat = 0.0
    for row in samples:
        m_hat = max(m_hat, max(row.upstream_norms))
    l_hat = 0.0
    if m_hat > 0.0:
        for row in samples:
            tail = 0.0
            for k in range(len(row.diffs) - 1, -1, -1):
                tail += row.diffs[k]
                if tail > 0.0:
                    l_hat = max(l_hat, row.raw_fwd[k] / (m_hat * tail))
    return l_hat, m_hat


def lemma1_report(samples, L: float, M: float) -> dict:
    """Measured forward-snapshot deviations against the L*M bound (theory.py:123-151)."""
    rows = []
    holds = 0
    for row in samples:
        rhs = lemma_bound_rhs(L, M, row.diffs)
        ok = all(lhs <= r for lhs, r in zip(row.raw_fwd, rhs))
        holds += ok
        rows.append({"batch_index": row.batch_index, "measured": list(row.raw_fwd), "bound": rhs, "holds": ok})
    return {"L": L, "M": M, "samples": len(rows), "holds_fraction": (holds / len(rows)) if rows else 1.0,
            "rows": rows}
