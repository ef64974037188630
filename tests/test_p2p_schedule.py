"""The symmetric diagonal-block schedule of the P2P pair kernel (paper_1204_3105_b200/csrc/p2p.cu).

Within a diagonal near block (t, t) in self mode (reading D16: the pair (i, i) is excluded),
the kernel walks row steps of 8 rows and column halves of 16 and, for a row step
[rc, rc + 8) and a half starting at a:
  * skips the half when a + 15 < rc,
  * evaluates it one-sided (rows only) when a <= rc + 7,
  * evaluates it symmetrically (rows + reactions) otherwise.
Every ordered pair (i, j), i != j, must be counted exactly once.  This enumerates the rule
for every leaf occupancy the kernel takes on that path (n <= P2P_S = 160).
"""
import pytest


def schedule_counts(n, rows=8, half=16):
    cnt = {}
    for rc in range(0, n, rows):
        for a in range(0, n, half):
            if a + half - 1 < rc:
                continue
            straddle = a <= rc + rows - 1
            for i in range(rc, min(rc + rows, n)):
                for j in range(a, min(a + half, n)):
                    if i == j:
                        continue
                    cnt[(i, j)] = cnt.get((i, j), 0) + 1
                    if not straddle:
                        cnt[(j, i)] = cnt.get((j, i), 0) + 1
    return cnt


@pytest.mark.parametrize("n", list(range(1, 41)) + [63, 64, 65, 97, 128, 159, 160])
def test_each_ordered_pair_once(n):
    cnt = schedule_counts(n)
    assert all(v == 1 for v in cnt.values())
    assert len(cnt) == n * (n - 1)


def test_symmetric_work_fraction():
    # the schedule evaluates well under the n^2 of a one-sided diagonal block at leaf sizes
    # of the benchmark workloads (64 .. 143 points per leaf)
    for n in (64, 143):
        evaluated = 0
        for rc in range(0, n, 8):
            for a in range(0, n, 16):
                if a + 15 < rc:
                    continue
                evaluated += min(8, n - rc) * min(16, n - a)
        assert evaluated < 0.7 * n * n
