"""GPU parity of contention on realised orders (reading R36:
adaptis_eval_contended / adaptis_search_contended) against the oracle
(oracle.contention.simulate_realised_contended: the event loop's realised
order executed by the R34 engine simulator): status, makespan and peak of
every candidate, and the argmin, on cfg1, random small spaces (latencies up
to 200 ticks so that transfers queue) and a cfg3 sample."""
import numpy as np
import pytest

from oracle import contention as CT
from oracle import oracle as O
from paper_2509_23722_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2509_23722_b200 import adaptis as A
    c = A.Context(0)
    yield c
    c.close()


def _want(pr, sp, indices):
    out = {"status": [], "makespan": [], "peak_mem": []}
    for i in indices:
        pl = O.decode(pr, sp, int(i))
        # the full cut list [0, ..., L]: an invalid BALL decode's interior cuts can
        # themselves start at 0 and end at L
        r = CT.simulate_realised_contended(pr, pl["v"], pl["placement"], pl["policy"], pl["cuts"])
        for k in out:
            out[k].append(r[k])
    return {k: np.asarray(v) for k, v in out.items()}


def _compare(got, want, where):
    for k in ("status", "makespan", "peak_mem"):
        g, w = np.asarray(got[k]), want[k]
        if k == "peak_mem":  # reported for status 0 / 2 only
            sel = np.isin(want["status"], (0, 2))
            g, w = g[sel], w[sel]
        bad = np.nonzero(g != w)[0]
        assert bad.size == 0, "%s %s mismatch at %s: gpu %s oracle %s" % (where, k, bad[:8], g[bad[:8]], w[bad[:8]])


def test_contended_cfg1_exhaustive_and_argmin(ctx):
    pr, sp = W.config(1)
    pr.comm = pr.comm * 50  # slow links: transfers queue on the engines
    prep = ctx.prepare(pr, sp)
    N = O.space_size(pr, sp)
    got = prep.eval_contended(0, N)
    want = _want(pr, sp, range(N))
    _compare(got, want, "cfg1")
    ok = want["status"] == 0
    best = int(np.nonzero(ok & (want["makespan"] == want["makespan"][ok].min()))[0][0])
    b = prep.search_contended()
    assert (b["index"], b["makespan"]) == (best, int(want["makespan"][best]))
    # contention changes some results against pure latency
    plain = O.eval_indices(pr, sp, range(N))
    assert np.any(np.asarray(plain["makespan"])[ok] != want["makespan"][ok])


@pytest.mark.parametrize("seed", [3, 4])
def test_contended_random_spaces(ctx, seed):
    """Spaces of up to 300 candidates whole (results and argmin), larger ones on
    a seeded block of 150 (the R34 oracle is pure Python)."""
    from test_gpu_parity import _random_spaces
    whole = 0
    for pr, sp in _random_spaces(seed, 8, cmax=200):
        N = O.space_size(pr, sp)
        prep = ctx.prepare(pr, sp)
        first = 0 if N <= 300 else int(np.random.default_rng(seed).integers(0, N - 150))
        count = N if N <= 300 else 150
        got = prep.eval_contended(first, count)
        want = _want(pr, sp, range(first, first + count))
        _compare(got, want, "p=%d m=%d" % (pr.p, pr.m))
        if N > 300:
            continue
        whole += 1
        ok = want["status"] == 0
        b = prep.search_contended()
        if ok.any():
            best = int(np.nonzero(ok & (want["makespan"] == want["makespan"][ok].min()))[0][0])
            assert (b["index"], b["makespan"]) == (best, int(want["makespan"][best]))
        else:
            assert b["index"] == O.UINT64_MAX
    assert whole > 0


def test_contended_cfg3_sample(ctx):
    pr, sp = W.config(3)
    pr.comm = pr.comm * 100
    prep = ctx.prepare(pr, sp)
    N = O.space_size(pr, sp)
    rng = np.random.default_rng(9)
    for first in [0] + [int(x) for x in rng.integers(0, N - 64, 3)]:
        got = prep.eval_contended(first, 64)
        _compare(got, _want(pr, sp, range(first, first + 64)), "cfg3@%d" % first)
