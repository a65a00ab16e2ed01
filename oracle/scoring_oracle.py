"""CPU restatement of the reference's scoring functions (TEST INFRASTRUCTURE).

Only tests/ import this module; it is the parity checker of the GPU oracle-WER
kernel (paper_1804_03243_b200/csrc/lb_scoring.cuh), pinned to the reference's
own outputs by tests/golden/scoring.npz (tests/golden/make_scoring_golden.py).

  wer              scoring.py:24-58   edit-distance counts, ties: sub > ins > del
  oracle_wer       scoring.py:66-114  deletion closure + arc relaxation swept to a
                                      fixpoint (vectorised over arcs per sweep: the
                                      fixpoint is the unique shortest-path table)
  lattice_density  scoring.py:121-130 arcs per frame
"""

from __future__ import annotations

import numpy as np


def wer(hyp, ref):
    """(substitutions, insertions, deletions), scoring.py:24-58."""
    if len(ref) == 0:
        raise ValueError("reference word sequence is empty")
    h, r = len(hyp), len(ref)
    d = np.zeros((h + 1, r + 1), dtype=np.int64)
    d[:, 0] = np.arange(h + 1)
    d[0, :] = np.arange(r + 1)
    for i in range(1, h + 1):
        for j in range(1, r + 1):
            d[i, j] = min(d[i - 1, j - 1] + (hyp[i - 1] != ref[j - 1]), d[i - 1, j] + 1, d[i, j - 1] + 1)
    subs = ins = dels = 0
    i, j = h, r
    while i > 0 or j > 0:
        if i > 0 and j > 0 and d[i, j] == d[i - 1, j - 1] + (hyp[i - 1] != ref[j - 1]):
            subs += int(hyp[i - 1] != ref[j - 1])
            i, j = i - 1, j - 1
        elif i > 0 and d[i, j] == d[i - 1, j] + 1:
            ins += 1
            i -= 1
        else:
            dels += 1
            j -= 1
    return subs, ins, dels


def oracle_wer(num_nodes, start, final_ids, from_, to, olabel, ref):
    """Fewest word errors over complete lattice paths (scoring.py:66-114);
    None when no complete path exists."""
    if len(ref) == 0:
        raise ValueError("reference word sequence is empty")
    n, r = int(num_nodes), len(ref)
    inf = np.iinfo(np.int64).max // 2
    best = np.full((n, r + 1), inf, dtype=np.int64)
    best[start, 0] = 0
    ref = np.asarray(ref, dtype=np.int64)
    frm, to, ol = (np.asarray(x, dtype=np.int64) for x in (from_, to, olabel))
    eps, wrd = ol == 0, ol != 0

    def close():
        for j in range(1, r + 1):
            np.minimum(best[:, j], best[:, j - 1] + 1, out=best[:, j])

    for _ in range(n * (r + 1) + 2):
        close()
        before = best.copy()
        np.minimum.at(best, to[eps], best[frm[eps]])
        np.minimum.at(best, to[wrd], best[frm[wrd]] + 1)
        cost = best[frm[wrd], :r] + (ol[wrd][:, None] != ref[None, :])
        sub = best[:, 1:].copy()
        np.minimum.at(sub, to[wrd], cost)
        best[:, 1:] = np.minimum(best[:, 1:], sub)
        close()
        if np.array_equal(best, before):
            break
    res = int(min(best[int(f), r] for f in final_ids)) if len(final_ids) else inf
    return None if res >= inf else res


def lattice_density(num_arcs, num_frames):
    return num_arcs / float(num_frames)
