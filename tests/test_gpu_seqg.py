"""The sequential GREEDY kernel (adaptis_seqg.cu: one exact event loop per
thread) against the oracle, and its dispatch. GREEDY segments with int32
ticks, p in {2, 4, 8, 16}, m <= 255 whose state fits run on it; everything it
cannot hold exactly (K = 2 arrival slots per edge) is re-run by the
global-ring kernel."""
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


def test_seq_runs_the_greedy_segments(ctx):
    pr, sp = W.config(3)
    idx = np.arange(0, O.space_size(pr, sp), 9973, dtype=np.uint64)  # every segment
    ctx.prepare(pr, sp).eval_indices(idx)
    info = [li for li in ctx.launch_info() if li["candidates"]]
    assert len(info) == 10
    assert any(li["kernel"] == 1 for li in info)
    for li in info:
        assert (li["kernel"] == 1) == (li["policy"] == W.GREEDY), li


@pytest.mark.parametrize("cid", [3, 4, 5])
def test_seq_blocks_equal_oracle(ctx, cid):
    """Every GREEDY (group, combo) segment of the config: the first 1024
    candidates (the seed neighbourhood) and a seeded random block."""
    pr, sp = W.config(cid)
    N = O.space_size(pr, sp)
    rng = np.random.default_rng(4242 + cid)
    base = 0
    seen = 0
    for g in sp.groups:
        one = W.Space([g])
        n_g = O.space_size(pr, one)
        k = 0
        for c in range(6):
            if not (g.combo_mask >> c) & 1 or O.combo(g.v, c) is None:
                continue
            seg = W.Space([W.Group(g.v, g.part_mode, g.radius, g.seed_cuts, 1 << c)])
            n_s = O.space_size(pr, seg)
            if O.combo(g.v, c)[1] == W.GREEDY and (cid != 5 or seen < 3):
                for first in (base + k, base + k + int(rng.integers(0, max(1, n_s - 1024)))):
                    cnt = min(1024 if cid != 5 else 128, N - first)
                    got = ctx.eval_batch(pr, sp, first, cnt)
                    _compare(got, O.eval_indices(pr, sp, range(first, first + cnt)),
                             "cfg%d v=%d combo %d @%d" % (cid, g.v, c, first))
                seen += 1
            k += n_s
        base += n_g
    assert seen > 0


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_seq_random_spaces_with_overflow(ctx, seed):
    """Random problems with latencies up to 200 ticks against task durations of
    1-9: many edges hold more than K future arrivals, so candidates overflow and
    are re-run by the exact global-ring kernel; results equal the oracle."""
    from test_gpu_parity import _random_spaces
    before = ctx.fallback_count
    for pr, sp in _random_spaces(seed, 10, cmax=200):
        N = O.space_size(pr, sp)
        got = ctx.eval_batch(pr, sp, 0, N)
        _compare(got, O.eval_indices(pr, sp, range(N)), "p=%d m=%d" % (pr.p, pr.m))
        b = ctx.search(pr, sp)
        ob = O.search(pr, sp, prune=False)
        if ob["index"] != O.UINT64_MAX:
            assert (b["index"], b["makespan"]) == (ob["index"], ob["makespan"])
    assert ctx.fallback_count > before


def test_lane_kernel_still_exact_when_seq_disabled(monkeypatch):
    """ADAPTIS_NO_SEQ=1 keeps GREEDY on the lane-per-device kernel (used for
    int64 / fp32 ticks, other p, m > 255 and reports): same winner."""
    from paper_2509_23722_b200 import adaptis as A
    from test_gpu_goldens import golden_argmin
    monkeypatch.setenv("ADAPTIS_NO_SEQ", "1")
    c = A.Context(0)
    try:
        pr, sp = W.config(4)
        b = c.search(pr, sp)
        g = golden_argmin(4)
        assert (b["index"], b["makespan"]) == (g["index"], g["makespan"])
        assert all(li["kernel"] != 1 for li in c.launch_info())
    finally:
        c.close()


def test_seq_wide_stage_durations_fall_back(ctx):
    """The sequential kernel keeps t_F and t_B of a stage in 16 bits: cfg1 with
    F/B costs scaled x12 has stages on both sides of 2^16 ticks; the wide ones
    are re-run by the global-ring kernel and every result equals the oracle."""
    import copy
    pr, sp = W.config(1)
    pr = copy.copy(pr)
    pr.t_f = np.asarray(pr.t_f) * 12
    pr.t_b = np.asarray(pr.t_b) * 12
    N = O.space_size(pr, sp)
    before = ctx.fallback_count
    got = ctx.eval_batch(pr, sp, 0, N)
    _compare(got, O.eval_indices(pr, sp, range(N)), "cfg1 x12")
    assert ctx.fallback_count > before
    assert any(li["kernel"] == 1 for li in ctx.launch_info())
    b = ctx.search(pr, sp)
    ob = O.search(pr, sp, prune=False)
    assert (b["index"], b["makespan"]) == (ob["index"], ob["makespan"])
