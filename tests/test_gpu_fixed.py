"""The static-order kernel (adaptis_fixed.cu: GPIPE / ONEF1B / ZB as one
topological order of F/B entries per segment, one thread per candidate)
against the oracle, and its dispatch. Segments it cannot take (int64 / fp32
ticks, p > 16, traces, reports, explicit plans) stay on the lane kernels,
which ADAPTIS_NO_FIXED=1 selects for every fixed-order segment."""
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


def _compare(got, want, where=""):
    for k in ("status", "makespan", "peak_mem"):
        g, w = np.asarray(got[k]), np.asarray(want[k])
        bad = np.nonzero(g != w)[0]
        assert bad.size == 0, "%s %s mismatch at %s: gpu %s oracle %s" % (
            where, k, bad[:10], g[bad[:10]], w[bad[:10]])
    ok = np.asarray(want["status"]) == 0
    assert np.all(np.abs(np.asarray(got["bubble"])[ok] - np.asarray(want["bubble"])[ok]) <= 1e-6)


def test_fixed_runs_the_fixed_order_segments(ctx):
    pr, sp = W.config(3)
    idx = np.arange(0, O.space_size(pr, sp), 9973, dtype=np.uint64)  # every segment
    ctx.prepare(pr, sp).eval_indices(idx)
    info = [li for li in ctx.launch_info() if li["candidates"]]
    assert len(info) == 10
    for li in info:
        assert li["kernel"] == (1 if li["policy"] == W.GREEDY else 2), li


def _segments(pr, sp):
    """(first index, size, v, combo) of every (group, combo) segment."""
    base = 0
    for g in sp.groups:
        k = 0
        for c in range(6):
            if not (g.combo_mask >> c) & 1 or O.combo(g.v, c) is None:
                continue
            seg = W.Space([W.Group(g.v, g.part_mode, g.radius, g.seed_cuts, 1 << c)])
            n_s = O.space_size(pr, seg)
            yield base + k, n_s, g.v, c
            k += n_s
        base += O.space_size(pr, W.Space([g]))


@pytest.mark.parametrize("cid", [2, 3, 4, 5])
def test_fixed_blocks_equal_oracle(ctx, cid):
    """Every GPIPE / ONEF1B / ZB segment: the first candidates (the seed
    neighbourhood) and a seeded random block, element by element."""
    pr, sp = W.config(cid)
    rng = np.random.default_rng(5151 + cid)
    seen = 0
    cnt = 512 if cid != 5 else 64
    for first, n_s, v, c in _segments(pr, sp):
        if O.combo(v, c)[1] == W.GREEDY:
            continue
        for f in (first, first + int(rng.integers(0, max(1, n_s - cnt)))):
            n = min(cnt, first + n_s - f)
            got = ctx.eval_batch(pr, sp, f, n)
            _compare(got, O.eval_indices(pr, sp, range(f, f + n)), "cfg%d v=%d combo %d @%d" % (cid, v, c, f))
        seen += 1
    assert seen > 0


@pytest.mark.parametrize("seed", [21, 22, 23])
def test_fixed_random_spaces_with_caps(ctx, seed):
    """Random problems (p = 1..8, caps that bind, latencies up to 200 ticks):
    the ZB W-fill's memory rule and the fused orders' closed-form peak decide
    many candidates; every result and the argmin equal the oracle."""
    from test_gpu_parity import _random_spaces
    for pr, sp in _random_spaces(seed, 10, cmax=200):
        N = O.space_size(pr, sp)
        got = ctx.eval_batch(pr, sp, 0, N)
        _compare(got, O.eval_indices(pr, sp, range(N)), "p=%d m=%d" % (pr.p, pr.m))
        b = ctx.search(pr, sp)
        ob = O.search(pr, sp, prune=False)
        if ob["index"] != O.UINT64_MAX:
            assert (b["index"], b["makespan"]) == (ob["index"], ob["makespan"])


def test_lane_kernels_still_exact_when_fixed_disabled(monkeypatch):
    """ADAPTIS_NO_FIXED=1 keeps the fixed orders on the lane-per-device
    kernels (used for int64 / fp32 ticks, p > 16, traces and reports)."""
    from paper_2509_23722_b200 import adaptis as A
    from test_gpu_goldens import golden_argmin
    monkeypatch.setenv("ADAPTIS_NO_FIXED", "1")
    c = A.Context(0)
    try:
        pr, sp = W.config(2)
        b = c.search(pr, sp)
        g = golden_argmin(2)
        assert (b["index"], b["makespan"]) == (g["index"], g["makespan"])
        assert all(li["kernel"] != 2 for li in c.launch_info())
    finally:
        c.close()


def test_fixed_large_sv_instances_equal_oracle(monkeypatch):
    """ADAPTIS_FIXED_MINW=1 puts cfg5's p = 16, v = 4 (S = 64) ZB and ONEF1B
    segments on the static-order kernel (by default they stay on the lane
    kernel for occupancy): blocks of both equal the oracle."""
    from paper_2509_23722_b200 import adaptis as A
    monkeypatch.setenv("ADAPTIS_FIXED_MINW", "1")
    pr, sp = W.config(5)
    c = A.Context(0)
    try:
        seen = 0
        for first, n_s, v, cb in _segments(pr, sp):
            if v != 4 or O.combo(v, cb)[1] not in (W.ZB, W.ONEF1B):
                continue
            n = min(48, n_s)
            got = c.eval_batch(pr, sp, first, n)
            assert all(li["kernel"] == 2 for li in c.launch_info() if li["candidates"])
            _compare(got, O.eval_indices(pr, sp, range(first, first + n)), "cfg5 v=4 combo %d" % cb)
            seen += 1
        assert seen == 2
    finally:
        c.close()
