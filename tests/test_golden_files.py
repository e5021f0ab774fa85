"""The oracle-generated golden files (tests/make_goldens.py) on the CPU: every
line well formed, and every cluster's statistics inside the bounds the paper
fixes for Alg. 1:

* |F_0| = the cluster's sources (R1 seeding): 1 <= |F_0| <= 64;
* a vertex is in at most d + 1 frontiers of a cluster, so
  sum_i |F_i| <= (d + 1) * n and sum_i E_i <= (d + 1) * m_reach, where m_reach
  (the summed degree of the reached vertices) is at most the arc count;
* the per-round records sum to the totals, and every recorded frontier is
  non-empty until the last round (the loop runs while F_i is non-empty,
  P:713);
* cluster ids are unique and below the selection size of the header.

These pin the stored values to the paper's invariants at full size, and
guard the files against truncated or duplicated lines.
"""
import json
import os

import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CONFIGS = ["c1_er", "c2_rmat20", "c3_rmat24", "c4_grid", "c5_knn"]


def read(name):
    path = os.path.join(GOLDEN, f"{name}.golden.txt")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    text = open(path).read()
    assert text.endswith("\n"), "last line truncated"
    lines = text.splitlines()
    header = json.loads(lines[0][2:])
    return header, [ln for ln in lines[1:] if ln.strip() and not ln.startswith("#")]


@pytest.mark.parametrize("name", CONFIGS)
def test_golden_lines_within_paper_bounds(name):
    header, lines = read(name)
    n, arcs, C, d = header["n"], header["arcs"], header["clusters"], header["d"]
    seen = set()
    for ln in lines:
        f = [int(x) for x in ln.split()]
        assert len(f) >= 6, ln[:80]
        c, R, sF, sE, mr = f[:5]
        assert 0 <= c < C and c not in seen, c
        seen.add(c)
        assert 1 <= R and 0 <= mr <= arcs, c
        assert 1 <= sF <= (d + 1) * n, c
        assert sE <= (d + 1) * mr, c
        if len(f) > 6:
            rounds = f[6:]
            assert len(rounds) == 2 * R, c
            F, E = rounds[0::2], rounds[1::2]
            assert sum(F) == sF and sum(E) == sE, c
            assert 1 <= F[0] <= 64, c
            assert all(x > 0 for x in F), c
    assert seen, "empty golden"
