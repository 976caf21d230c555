"""Host-side invariants of the tensor-core Cholesky's task DAG (csrc/vba_chol.cu
chol_plan_tasks_tc, exported as vba_chol_plan): the factorisation np.linalg.solve stands
for (solver.py:287) runs as one chain task (POTRF -> TRSM -> SYRK of every step) plus
left-looking tile tasks claimed in list order by persistent CTAs that spin on flags, so the
list must produce every tile exactly once and must never let a claimed task wait on work that
can only start later.  No GPU needed.
"""
import ctypes as C

import numpy as np
import pytest

from paper_2512_02293_b200 import _lib as L

T_TRSM, T_CHAIN, T_TILE, T_CONV, T_PREP = 1, 6, 7, 8, 9
SYRK_TARGET, TILE_TRSM, OPERAND = 0, 1, 2


def _plan(nt):
    lib = L.load()
    n = lib.vba_chol_plan(nt, None, 0)
    assert n >= 0
    buf = (C.c_int32 * (5 * max(n, 1)))()
    assert lib.vba_chol_plan(nt, buf, n) == n
    return np.frombuffer(buf, dtype=np.int32)[: 5 * n].reshape(n, 5)


def test_bad_arguments():
    lib = L.load()
    assert lib.vba_chol_plan(-1, None, 0) == L.VBA_E_INVALID
    assert lib.vba_chol_plan(4, None, 3) == L.VBA_E_INVALID


@pytest.mark.parametrize("nt", [1, 2, 3, 4, 5, 8, 15, 60, 148])
def test_tc_cholesky_plan_invariants(nt):
    P = _plan(nt)
    assert P[0, 0] == T_CHAIN and int((P[:, 0] == T_CHAIN).sum()) == 1
    assert set(P[:, 0].tolist()) <= {T_TRSM, T_CHAIN, T_TILE, T_CONV, T_PREP}

    # producers: L_ij (i >= j+2) by a TRSM (j = 0) or a TILE in TRSM mode; the chain makes
    # L_{j+1,j} and Linv_jj at its step j
    prod, operand, syrk = {}, {}, {}
    for q, (t, i, j, k, m) in enumerate(P.tolist()):
        if t == T_TRSM:
            assert j == 0 and i >= 2 and (i, j) not in prod
            prod[(i, j)] = q
        elif t == T_TILE:
            if m == TILE_TRSM:
                assert i >= j + 2 and k == j and (i, j) not in prod
                prod[(i, j)] = q
            elif m == OPERAND:
                assert i == j + 1 and k == j and (i, j) not in operand
                operand[(i, j)] = q
            else:
                assert m == SYRK_TARGET and i == j and k == j - 1 and (i, j) not in syrk
                syrk[(i, j)] = q
    assert set(prod) == {(i, j) for j in range(nt) for i in range(j + 2, nt)}
    assert set(operand) == {(j + 1, j) for j in range(nt - 1)}
    assert set(syrk) == {(j, j) for j in range(2, nt)}
    conv = [q for q, t in enumerate(P[:, 0].tolist()) if t == T_CONV]
    prep = [q for q, t in enumerate(P[:, 0].tolist()) if t == T_PREP]
    assert sorted(P[conv, 1].tolist()) == list(range(nt))
    # the folded solve matrices: every (k, kind) whose neighbour tile exists, exactly once
    want = {(k, kind) for k in range(nt) for kind in range(5)
            if not ((kind == 1 and k < 1) or (kind == 2 and k < 2) or (kind == 3 and k + 1 >= nt)
                    or (kind == 4 and k + 2 >= nt))}
    assert sorted(map(tuple, P[prep][:, 1:3].tolist())) == sorted(want)
    assert conv + prep == list(range(len(P) - nt - len(prep), len(P)))   # the list ends with them

    # every input of a task is made earlier in claim order or by the chain; need[q] = the
    # latest chain step task q waits for
    need = np.full(len(P), -1)

    def src(i, m, q):   # L_im for a task at position q
        if i == m + 1:
            return m                                     # chain step m
        assert prod[(i, m)] < q, (i, m, q)
        return need[prod[(i, m)]]

    for q, (t, i, j, k, m) in enumerate(P.tolist()):
        if t == T_TRSM:
            need[q] = j                                  # Linv_jj
        elif t == T_TILE:
            w = -1
            for c in range(k):
                w = max(w, src(i, c, q), src(j, c, q))
            if m == TILE_TRSM:
                w = max(w, j)
            need[q] = w
        elif t == T_CONV:
            need[q] = k                                  # Linv_kk, L_{k+1,k}
        elif t == T_PREP:                                # CONV(i) (+ CONV(i-1) or a TRSM tile)
            kk, kind = i, j
            need[q] = kk
            if kind == 2:
                assert prod[(kk, kk - 2)] < q
            if kind == 4:
                assert prod[(kk + 2, kk)] < q
    # chain step s waits for its operand (s+1, s) and SYRK target (s+1, s+1); no task claimed
    # before them may wait for a chain step beyond s (else every CTA could end up spinning)
    for s in range(nt - 1):
        gate = max(operand[(s + 1, s)], syrk.get((s + 1, s + 1), 0))
        assert need[operand[(s + 1, s)]] < s + 1 and need[syrk.get((s + 1, s + 1), 0)] <= s
        assert need[1:gate + 1].max(initial=-1) <= s, s
