"""Frozen input fixtures ("freeze the generated tables as test
fixtures ... parity then never depends on two RNG implementations agreeing").

tests/golden/tables_cfg{1..5}.json were written by tools/freeze_tables.py from
the seeded input generator alone. These tests check that the generator still
reproduces them, that they follow the §8(d) recipe, and that the canonical
space sizes of the configs are the ones SURVEY §8(d) lists.
"""
import json
import os

import pytest

from paper_2509_23722_b200 import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")
COLS = ("t_f", "t_b", "t_w", "act", "stash", "weight", "grad", "comm")
# SURVEY §8(d) config table, column N (exact values of the canonical space, R19)
SPACE_N = {1: 244, 2: 4_272_048, 3: 182_684_682, 4: 145_990_662, 5: 949_873_416}
# SURVEY §8(d) kind table: t_F, t_B, t_W (ticks), act, stash, weight, grad (MiB)
KIND_BASE = {
    "E": (60, 60, 120, 32, 16, 1000, 2000), "D": (1000, 1000, 900, 640, 320, 400, 800),
    "F": (1100, 1100, 1000, 700, 350, 450, 900), "X": (1500, 1500, 1350, 900, 450, 800, 1600),
    "M": (700, 700, 600, 320, 160, 300, 600), "A": (600, 600, 400, 400, 200, 150, 300),
    "P": (500, 500, 500, 300, 150, 250, 500), "H": (2600, 2600, 2600, 2048, 1024, 1000, 2000),
}


def load(cid):
    with open(os.path.join(GOLD, "tables_cfg%d.json" % cid)) as f:
        return json.load(f)


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_generator_reproduces_fixture(cid):
    fx = load(cid)
    pr, sp = W.config(cid)
    assert (pr.L, pr.p, pr.m, pr.cap) == (fx["L"], fx["p"], fx["m"], fx["cap"])
    for c in COLS:
        assert [int(x) for x in getattr(pr, c)] == fx["columns"][c], c
    assert [(g.v, g.part_mode, g.radius, g.combo_mask) for g in sp.groups] == \
        [(g["v"], g["part_mode"], g["radius"], g["combo_mask"]) for g in fx["groups"]]


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_fixture_follows_recipe(cid):
    """Every row is a §8(d) kind scaled by a jitter in [0.97, 1.03], rounded."""
    fx = load(cid)
    cols = fx["columns"]
    mib = 1 << 20
    for l in range(fx["L"]):
        vals = [cols["t_f"][l], cols["t_b"][l], cols["t_w"][l]] + \
               [cols[c][l] / mib for c in ("act", "stash", "weight", "grad")]
        fits = [k for k, base in KIND_BASE.items()
                if all(0.97 * b - 1 <= v <= 1.03 * b + 1 for v, b in zip(vals, base))]
        assert fits, (cid, l, vals)
        assert all(x >= 1 for x in vals[:3])
    assert cols["comm"][-1] == 0 or fx["L"] == 8  # no boundary after the LM head
    assert all(35 <= c <= 45 for c in cols["comm"][:-1]) or cid == 1


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_space_size_matches_survey(cid):
    from oracle import oracle as O
    pr, sp = W.config(cid)
    assert O.space_size(pr, sp) == SPACE_N[cid]
