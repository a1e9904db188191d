"""GPU parity at the edges of the boundary's ranges (include/adaptis.h):
p = 32 (one candidate per warp), S = 64, v = 3 and 4 with odd p, S = L,
large L (prefix table near the shared-memory limit), an L too large for it
(clean EINVAL), empty and boundary ranges, and a cap of 0. Every case is
compared element by element with the oracle."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2509_23722_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2509_23722_b200 import adaptis as A
    c = A.Context(0)
    yield c
    c.close()


def _compare(got, want, where):
    for k in ("status", "makespan", "peak_mem"):
        g, w = np.asarray(got[k]), np.asarray(want[k])
        bad = np.nonzero(g != w)[0]
        assert bad.size == 0, "%s %s mismatch at %s: gpu %s oracle %s" % (
            where, k, bad[:8], g[bad[:8]], w[bad[:8]])


def _exhaustive(ctx, pr, sp, where, search=True):
    N = O.space_size(pr, sp)
    got = ctx.eval_batch(pr, sp, 0, N)
    want = O.eval_indices(pr, sp, range(N))
    _compare(got, want, where)
    if search:
        b = ctx.search(pr, sp)
        ob = O.search(pr, sp, prune=False)
        if ob["index"] == O.UINT64_MAX:
            assert b["status"] == 2
        else:
            assert (b["index"], b["makespan"]) == (ob["index"], ob["makespan"]), where
    return N


CASES = [
    # (p, m, L, groups, cap)
    (32, 32, 70, [(1, 1, 0xF), (2, 1, 0x3F)], None),   # one slot per warp, S = 32 and 64
    (16, 16, 64, [(4, 2, 0x3F)], None),                # S = 64 = L: one valid partition
    (7, 14, 30, [(3, 2, 0x3F), (1, 2, 0xF)], None),    # v = 3, p not a power of two
    (3, 6, 12, [(4, 3, 0x3F)], None),                  # S = 12 = L
    (5, 10, 40, [(2, 2, 0x3F), (4, 1, 0x3F)], 120),    # binding cap, v = 4
    (2, 1, 9, [(1, 3, 0xF)], None),                    # m = 1 < p
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_edge_shapes_exhaustive(ctx, case):
    p, m, L, groups, cap = CASES[case]
    rng = W.SplitMix64(777 + case)
    pr = W.random_problem(rng, L, p, m, tmax=9, cmax=4, bytes_max=6,
                          cap=W.INT64_MAX if cap is None else cap)
    sp = W.Space([W.Group(v, W.BALL, R, combo_mask=mask) for v, R, mask in groups])
    _exhaustive(ctx, pr, sp, "p=%d m=%d L=%d" % (p, m, L))


def test_large_L_prefix_table(ctx):
    """L = 2000 rows: a 96 KB prefix table per CTA (lower occupancy, same results)."""
    rng = W.SplitMix64(4242)
    pr = W.random_problem(rng, 2000, 4, 8, tmax=50, cmax=4, bytes_max=6)
    sp = W.Space([W.Group(1, W.BALL, 2, combo_mask=0xF), W.Group(2, W.BALL, 1, combo_mask=0x3F)])
    _exhaustive(ctx, pr, sp, "L=2000")


def test_L_beyond_shared_memory_is_einval(ctx):
    from paper_2509_23722_b200 import adaptis as A
    rng = W.SplitMix64(4343)
    pr = W.random_problem(rng, 6000, 2, 4, tmax=5, cmax=2, bytes_max=3)
    sp = W.Space([W.Group(1, W.BALL, 1, combo_mask=0x2)])
    with pytest.raises(A.AdaptisError) as e:
        ctx.eval_batch(pr, sp, 0, 3)
    assert e.value.status == A.EINVAL and "shared memory" in str(e.value)


def test_empty_and_boundary_ranges(ctx):
    from paper_2509_23722_b200 import adaptis as A
    pr, sp = W.config(1)
    N = O.space_size(pr, sp)
    got = ctx.eval_batch(pr, sp, N, 0)          # empty range at the end
    assert len(got["status"]) == 0
    got = ctx.eval_batch(pr, sp, N - 1, 1)      # last candidate
    want = O.eval_indices(pr, sp, [N - 1])
    _compare(got, want, "last")
    with pytest.raises(A.AdaptisError) as e:
        ctx.eval_batch(pr, sp, N, 1)
    assert e.value.status == A.EINVAL


def test_zero_cap_is_infeasible(ctx):
    pr, sp = W.config(1, cap=0)
    N = _exhaustive(ctx, pr, sp, "cap=0")
    got = ctx.eval_batch(pr, sp, 0, N)
    assert not np.any(np.asarray(got["status"]) == 0)
