"""The GS kernel's block decomposition (k_gs.cu) restated as a sequential numpy
model and checked against plain Gauss-Seidel (Eq. 13-14): with A symmetric and only its upper
32x32 tiles stored, row block kn's residual is assembled from
  row use   U(kn, J) x_J            J > kn owned by CTA rg, minus J = kn-1, kn-2 (mod T)
  scatter   U(kn-3, J)^T x_{kn-3}   J >= kn (J = kn into P_kn, J > kn into y_J, consumed at J)
  L, LL     A[kn, kn-1] x, A[kn, kn-2] x   (the leader)
  D         the in-block recurrence
with the column ownership pattern of dwc_internal.cuh (leader 3 of every 18 / 8 blocks).
Host-side logic only (no oracle, no GPU)."""
import numpy as np
import pytest

PAT = {1: [0], 2: [0, 1, 1, 0, 1, 1, 0, 1], 4: [0, 1, 2, 3, 1, 2, 3, 0, 1, 2, 3, 1, 2, 3, 0, 1, 2, 3]}


def own_of(g, J):
    p = PAT[g]
    return p[J % len(p)]


def segments(T, g, rg, kn):
    out = []
    row = [J for J in range(kn + 1, T) if own_of(g, J) == rg]
    while row and row[-1] in ((kn - 1) % T, (kn - 2) % T):
        row.pop()
    out += [(0, kn, J) for J in row]
    if kn >= 3:
        out += [(1, kn - 3, J) for J in range(kn, T) if own_of(g, J) == rg]
    return out


def gs_plain(A, b, sweeps):
    x = np.zeros(len(b))
    for _ in range(sweeps):
        for i in range(len(b)):
            x[i] = max(x[i] - (A[i] @ x - b[i]) / A[i, i], 0.0)
    return x


def gs_blocked(A, b, sweeps, g, B=4):
    n = len(b)
    T = n // B
    x = np.zeros(n)
    y = {}
    blk = lambda k: slice(B * k, B * k + B)
    for s in range(sweeps * T):
        kn = s % T
        P = np.zeros(B)
        for rg in range(g):
            for seg, I, J in segments(T, g, rg, kn):
                U = A[blk(I), blk(J)]
                if seg == 0:
                    P += U @ x[blk(J)]
                else:
                    v = U.T @ x[blk(I)]
                    if J == kn:
                        P += v
                    else:
                        y[(rg, J)] = y.get((rg, J), 0.0) + v
            if own_of(g, kn) == rg:
                P += y.pop((rg, kn), 0.0)
        for d in {(kn - 1) % T, (kn - 2) % T} - {kn}:
            P += A[blk(kn), blk(d)] @ x[blk(d)]
        D = A[blk(kn), blk(kn)]
        for r in range(B):
            i = B * kn + r
            x[i] = max(x[i] - (P[r] + D[r] @ x[blk(kn)] - b[i]) / A[i, i], 0.0)
    assert not any(np.any(v != 0) for v in y.values())   # every scatter consumed
    return x


@pytest.mark.parametrize("T,g", [(1, 1), (2, 1), (3, 1), (4, 1), (7, 2), (9, 4), (12, 2), (20, 4), (23, 4)])
def test_blocked_symmetric_gs_equals_plain_gs(T, g):
    rng = np.random.default_rng(T * 10 + g)
    n = 4 * T
    M = rng.standard_normal((n, n))
    A = M @ M.T / n + np.eye(n)
    b = rng.standard_normal(n)
    assert np.max(np.abs(gs_blocked(A, b, 4, g) - gs_plain(A, b, 4))) < 1e-12


def test_every_upper_tile_streamed_twice_per_sweep():
    """Each stored U(I, J), J > I, is used once as a row tile and once transposed (or via the
    leader's L / LL path) per sweep: the packed storage is read ~once from HBM, twice from L2."""
    for T, g in [(9, 4), (20, 4), (12, 2)]:
        uses = {}
        for kn in range(T):
            for rg in range(g):
                for seg, I, J in segments(T, g, rg, kn):
                    uses[(I, J, seg)] = uses.get((I, J, seg), 0) + 1
        for I in range(T):
            for J in range(I + 1, T):
                row = uses.get((I, J, 0), 0)
                tr = uses.get((I, J, 1), 0)
                by_leader_row = J in ((I - 1) % T, (I - 2) % T)
                by_leader_tr = J - I in (1, 2)
                assert row == (0 if by_leader_row else 1), (T, g, I, J)
                assert tr == (0 if by_leader_tr else 1), (T, g, I, J)
