"""ORACLE (test infrastructure only): CPU restatement of the reference's
process-layout model, /root/reference/proj/include/bfly/layout.hpp.

Only tests/ import this module; the product (paper_2002_03400_b200) never
does.  Pinned against the reference itself through tests/golden/layout.npz
(written by tests/golden/make_golden.py from oracle/_ref, i.e. layout.hpp
compiled unmodified).

kinds: 0 column, 1 row, 2 hybrid (layout_kind, layout.hpp:8).
"""
from __future__ import annotations

import numpy as np

COLUMN, ROW, HYBRID = 0, 1, 2


def log_p(p: int) -> int:
    """LayoutSpec::log_p (layout.hpp:35-39)."""
    g = 0
    while (1 << (g + 1)) <= p:
        g += 1
    return g


def validate(kind: int, levels: int, rank: int, p: int) -> None:
    """LayoutSpec::validate (layout.hpp:41-48)."""
    if levels < 1:
        raise ValueError("levels >= 1 required")
    if rank < 1:
        raise ValueError("rank >= 1 required")
    if p < 1 or (p & (p - 1)) != 0:
        raise ValueError("process count must be a power of two")
    if p > (1 << levels):
        raise ValueError("process count must not exceed 2^L")
    if kind not in (COLUMN, ROW, HYBRID):
        raise ValueError("unknown layout kind")


def comm_cost(kind: int, levels: int, rank: int, p: int):
    """Closed-form CommCostReport (layout.hpp:70-88):
    [exchange_volume, exchange_msgs, alltoall_volume, alltoall_msgs]."""
    validate(kind, levels, rank, p)
    per_proc = rank * (1 << levels) / p
    g = log_p(p)
    exch = max(0, 2 * g - levels) if kind == HYBRID else g
    return [per_proc * exch, exch, per_proc, min((1 << levels) // p, p - 1)]


def bit_reverse(v: int, bits: int) -> int:
    """detail::bit_reverse (layout.hpp:92-96)."""
    out = 0
    for i in range(bits):
        out |= ((v >> i) & 1) << (bits - 1 - i)
    return out


def column_owner(L, g, level, tau, nu):
    """detail::column_owner (layout.hpp:101-104)."""
    label = (tau << (L - level)) | bit_reverse(nu, L - level)
    return label >> (L - g)


def row_owner(L, g, level, tau, nu):
    """detail::row_owner (layout.hpp:105-108)."""
    label = (nu << level) | bit_reverse(tau, level)
    return label >> (L - g)


def owners(kind: int, L: int, center: int, p: int) -> np.ndarray:
    """assign_ownership (layout.hpp:139-188) flattened as
    [u leaves | v leaves | R levels center..L-1 | W levels 1..center | cores],
    2^L entries each, flat block index tau*2^(L-l)+nu (butterfly.hpp:38-43)."""
    validate(kind, L, 1, p)
    g = log_p(p)
    nb = 1 << L
    u_col = kind != ROW
    v_row = kind != COLUMN
    uo = column_owner if u_col else row_owner
    vo = row_owner if v_row else column_owner
    out = [[uo(L, g, L, tau, 0) for tau in range(nb)], [vo(L, g, 0, 0, nu) for nu in range(nb)]]
    for l in range(center, L):
        out.append([uo(L, g, l, i >> (L - l), i & ((1 << (L - l)) - 1)) for i in range(nb)])
    for l in range(1, center + 1):
        out.append([vo(L, g, l, i >> (L - l), i & ((1 << (L - l)) - 1)) for i in range(nb)])
    out.append([vo(L, g, center, i >> (L - center), i & ((1 << (L - center)) - 1)) for i in range(nb)])
    return np.array(out, np.int32)


def simulated_tallies(kind: int, L: int, center: int, p: int, u_rank, v_rank, rows: int, cols: int):
    """simulated_parallel_apply's CommCostReport (layout.hpp:190-261) from the
    ownership maps and the block ranks: u_rank(l, tau, nu), v_rank(l, tau, nu)."""
    o = owners(kind, L, center, p)
    nb = 1 << L

    def w_at(l, tau, nu):
        return o[2 + (L - center) + (l - 1)][tau * (1 << (L - l)) + nu]

    def r_at(l, tau, nu):
        return o[2 + (l - center)][tau * (1 << (L - l)) + nu]

    def v_coef_owner(l, tau, nu):
        return o[1][nu] if l == 0 else w_at(l, tau, nu)

    def state(fn, l):
        return float(sum(fn(l, tau, nu) for tau in range(1 << l) for nu in range(1 << (L - l))))

    ev, em = 0.0, 0
    for l in range(1, center + 1):
        moved = any(v_coef_owner(l - 1, tau // 2, 2 * nu) != w_at(l, tau, nu)
                    or v_coef_owner(l - 1, tau // 2, 2 * nu + 1) != w_at(l, tau, nu)
                    for tau in range(1 << l) for nu in range(1 << (L - l)))
        if moved:
            em += 1
            ev += state(v_rank, l - 1) / p
    for l in range(center, L):
        def consumer(tau, nu):
            return o[0][tau] if l + 1 == L else r_at(l + 1, tau, nu)
        moved = any(r_at(l, tau // 2, 2 * nu) != consumer(tau, nu) or r_at(l, tau // 2, 2 * nu + 1) != consumer(tau, nu)
                    for tau in range(1 << (l + 1)) for nu in range(1 << (L - l - 1)))
        if moved:
            em += 1
            ev += state(u_rank, l) / p
    if kind == COLUMN:
        av = cols / p
    elif kind == ROW:
        av = rows / p
    else:
        av = state(u_rank, center) / p
    return [ev, em, av, min(nb // p, p - 1)]
