"""Argmin parity on all five configs against oracle-written goldens, and the
exact fallback path forced on.

tests/golden/argmin_cfg{1..5}.json are written by tools/oracle_argmin.py, which
imports only oracle/ and the seeded input generator: the oracle's exact
LB-pruned exhaustive search (SURVEY §8(c) Pins, "Search / argmin"; Eq. 1-2,
P:339-343, lowest-index ties R18). No value in them comes from the CUDA path.
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2509_23722_b200 import workloads as W

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden_argmin(cid, tag=""):
    path = os.path.join(GOLDEN, "argmin_cfg%d%s.json" % (cid, tag))
    if not os.path.exists(path):
        pytest.skip("no oracle golden %s (run tools/oracle_argmin.py)" % os.path.basename(path))
    with open(path) as f:
        return json.load(f)


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


@pytest.mark.parametrize("prune", [True, False], ids=["pruned", "unpruned"])
@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_config_argmin_equals_oracle_golden(ctx, cid, prune):
    """North star: bit-exact plans on all five configs. The GPU search (the
    pruned time-to-best-plan search and the unpruned throughput search) returns
    the oracle's exhaustive winner (index, makespan, plan), and counts exactly
    the oracle's invalid decodes (R19)."""
    g = golden_argmin(cid)
    pr, sp = W.config(cid)
    ctx.set_prune(prune)
    try:
        b = ctx.search(pr, sp)
    finally:
        ctx.set_prune(False)
    assert (b["index"], b["makespan"]) == (g["index"], g["makespan"])
    assert b["plan"]["cuts"] == g["plan"]["cuts"]
    assert (b["plan"]["v"], b["plan"]["placement"], b["plan"]["policy"]) == (
        g["plan"]["v"], g["plan"]["placement"], g["plan"]["policy"])
    assert b["n_candidates"] == g["n_total"]
    assert b["n_invalid"] == g["n_invalid"], (b["n_invalid"], g["n_invalid"])


def _random_spaces(seed, n):
    from test_gpu_parity import _random_spaces as rs
    return rs(seed, n)


def test_forced_fallback_matches_oracle(ctx, monkeypatch):
    """ADAPTIS_RING_K=2 makes the lane kernels' fixed-order shared-memory rings
    overflow on most candidates, so the exact fallback kernel (global rings of
    depth >= m, re-run from the overflow list) decides them: evaluations and
    searches still equal the oracle, and the fallback really ran."""
    monkeypatch.setenv("ADAPTIS_RING_K", "2")
    monkeypatch.setenv("ADAPTIS_NO_SEQ", "1")  # the lane-per-device kernels and their rings
    before = ctx.fallback_count
    pr, sp = W.config(1)
    got = ctx.eval_batch(pr, sp, 0, 244)
    _compare(got, O.eval_indices(pr, sp, range(244)), "cfg1 K=2")
    b = ctx.search(pr, sp)
    g = golden_argmin(1)
    assert (b["index"], b["makespan"]) == (g["index"], g["makespan"])
    pr, sp = W.config(2)
    for first in (0, 2_000_000):
        got = ctx.eval_batch(pr, sp, first, 4096)
        _compare(got, O.eval_indices(pr, sp, range(first, first + 4096)), "cfg2 K=2 @%d" % first)
    for pr, sp in _random_spaces(7, 12):
        N = O.space_size(pr, sp)
        got = ctx.eval_batch(pr, sp, 0, N)
        _compare(got, O.eval_indices(pr, sp, range(N)), "random K=2 p=%d m=%d" % (pr.p, pr.m))
        b = ctx.search(pr, sp)
        ob = O.search(pr, sp, prune=False)
        if ob["index"] != O.UINT64_MAX:
            assert (b["index"], b["makespan"]) == (ob["index"], ob["makespan"])
    assert ctx.fallback_count > before


def test_whole_shard_fallback_counts_once(ctx, monkeypatch):
    """More overflowed candidates than a segment's overflow list holds re-run the
    whole segment shard in fallback mode (the list capacity is forced down to
    4096 here). The winner still equals the oracle's, and the invalid count is
    the oracle's exactly: the re-run's counts replace the first pass's for that
    segment instead of adding to them."""
    monkeypatch.setenv("ADAPTIS_RING_K", "2")
    monkeypatch.setenv("ADAPTIS_OVERFLOW_CAP", "4096")
    monkeypatch.setenv("ADAPTIS_NO_SEQ", "1")  # the lane-per-device kernels and their rings
    g = golden_argmin(3)
    pr, sp = W.config(3)
    b = ctx.search(pr, sp)
    assert (b["index"], b["makespan"]) == (g["index"], g["makespan"])
    assert b["n_invalid"] == g["n_invalid"]
    assert max(li["fallback"] for li in ctx.launch_info()) > 4096


def test_eval_indices_fallback_matches_oracle(ctx, monkeypatch):
    """adaptis_eval_indices (explicit index positions) with the fallback forced:
    overflowed candidates are re-run from their recorded output slots (list
    mode); seeded-uniform cfg3 indices, the block around the oracle's winner and
    every candidate of random small spaces, element by element."""
    monkeypatch.setenv("ADAPTIS_RING_K", "1")
    monkeypatch.setenv("ADAPTIS_NO_SEQ", "1")  # the lane-per-device kernels and their rings
    before = ctx.fallback_count
    pr, sp = W.config(3)
    N = O.space_size(pr, sp)
    w = golden_argmin(3)["index"]
    idx = np.concatenate([np.random.default_rng(777).integers(0, N, 10_000),
                          np.arange(w - 5000, w + 5000)]).astype(np.uint64)
    got = ctx.prepare(pr, sp).eval_indices(idx)
    _compare(got, O.eval_indices(pr, sp, idx), "cfg3 uniform K=1")
    fb = [li["fallback"] for li in ctx.launch_info()]
    for pr2, sp2 in _random_spaces(8, 12):
        N2 = O.space_size(pr2, sp2)
        idx2 = np.random.default_rng(5).permutation(N2).astype(np.uint64)  # shuffled: no runs
        got = ctx.prepare(pr2, sp2).eval_indices(idx2)
        _compare(got, O.eval_indices(pr2, sp2, idx2), "random K=1 p=%d m=%d" % (pr2.p, pr2.m))
        fb += [li["fallback"] for li in ctx.launch_info()]
    assert ctx.fallback_count > before, fb
