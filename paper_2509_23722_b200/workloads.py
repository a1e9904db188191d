"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no stage sums, schedules,
seeds or counts): only the problem/space containers and the seeded layer-table
generator of DESIGN.md §"Input recipe": per-kind costs in ticks
(1 tick = 1 us) and bytes, each multiplied by a splitmix64 jitter in
[0.97, 1.03) and rounded to an integer.

Kind ratios follow the paper's model families (Table 3): dense
self-attention+FFN (Llama/Gemma), MLA + dense FFN / MLA + MoE (DeepSeek),
Mamba-2 / attention-only / MLP-only (Nemotron-H), and a heavy LM head
(P:121).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

MiB = 1 << 20
INT64_MAX = (1 << 63) - 1

# policies / placements / partition modes (numbering of include/adaptis.h)
GPIPE, ONEF1B, ZB, GREEDY = 0, 1, 2, 3
SEQ, INTERLEAVED, WAVE = 0, 1, 2
FULL, BALL = 0, 1

# kind: (t_F, t_B, t_W ticks; act, stash, weight, grad MiB; comm ticks after)
KINDS = {
    "E": (60, 60, 120, 32, 16, 1000, 2000, 40),        # embedding
    "D": (1000, 1000, 900, 640, 320, 400, 800, 40),    # dense SA + FFN
    "F": (1100, 1100, 1000, 700, 350, 450, 900, 40),   # MLA + dense FFN
    "X": (1500, 1500, 1350, 900, 450, 800, 1600, 40),  # MLA + MoE
    "M": (700, 700, 600, 320, 160, 300, 600, 40),      # Mamba-2
    "A": (600, 600, 400, 400, 200, 150, 300, 40),      # attention-only
    "P": (500, 500, 500, 300, 150, 250, 500, 40),      # MLP-only
    "H": (2600, 2600, 2600, 2048, 1024, 1000, 2000, 0),  # LM head (V ~ 128K)
}
COLUMNS = ("t_f", "t_b", "t_w", "act", "stash", "weight", "grad", "comm")


class SplitMix64:
    """splitmix64 (Steele, Lea, Flood 2014); the only RNG of the test inputs."""

    def __init__(self, seed: int):
        self.s = seed & 0xFFFFFFFFFFFFFFFF

    def next(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        return z ^ (z >> 31)

    def uniform(self) -> float:
        return (self.next() >> 11) * (1.0 / (1 << 53))


@dataclass
class Problem:
    """Profiled data + training configuration ("Input")."""
    t_f: np.ndarray
    t_b: np.ndarray
    t_w: np.ndarray
    act: np.ndarray
    stash: np.ndarray
    weight: np.ndarray
    grad: np.ndarray
    comm: np.ndarray
    p: int
    m: int
    cap: int = INT64_MAX
    tick_seconds: float = 1e-6
    tokens_per_microbatch: int = 4096
    name: str = ""
    cost_type: int = 0                   # 0: exact int64 ticks, 1: fp32-cost variant
    costs_f32: Optional[np.ndarray] = None  # fp32 variant: [4][L] t_f, t_b, t_w, comm

    def __post_init__(self):
        for c in COLUMNS:
            setattr(self, c, np.ascontiguousarray(np.asarray(getattr(self, c), dtype=np.int64)))
        if self.costs_f32 is not None:
            self.costs_f32 = np.ascontiguousarray(np.asarray(self.costs_f32, dtype=np.float32))

    @property
    def L(self) -> int:
        return int(self.t_f.shape[0])


@dataclass
class Group:
    v: int
    part_mode: int = FULL
    radius: int = 0
    seed_cuts: Optional[List[int]] = None
    combo_mask: int = 0x3F


@dataclass
class Space:
    groups: List[Group] = field(default_factory=list)


def table_from_kinds(pattern: str, seed: int) -> dict:
    """Layer table for a kind string, e.g. 'EDDXXMDH', with seeded jitter."""
    rng = SplitMix64(seed)
    cols = {c: [] for c in COLUMNS}
    for k in pattern:
        base = KINDS[k]
        for ci, c in enumerate(COLUMNS):
            jit = 0.97 + 0.06 * rng.uniform()
            scale = MiB if 3 <= ci <= 6 else 1
            cols[c].append(int(round(base[ci] * scale * jit)))
    cols["comm"][-1] = 0  # no boundary after the LM head
    return {c: np.array(v, dtype=np.int64) for c, v in cols.items()}


def cfg5_pattern(seed: int = 5) -> str:
    rng = SplitMix64(seed)
    cum = [("D", 0.40), ("X", 0.60), ("M", 0.85), ("A", 0.90), ("P", 1.0)]
    out = []
    for _ in range(128):
        u = rng.uniform()
        for k, c in cum:
            if u < c:
                out.append(k)
                break
    return "E" + "".join(out) + "H"


def cfg4_pattern() -> str:
    hidden, alt = [], 0
    for i in range(52):
        if i in (7, 20, 33, 46):
            hidden.append("A")
        else:
            hidden.append("M" if alt % 2 == 0 else "P")
            alt += 1
    return "E" + "".join(hidden) + "H"


PATTERNS = {
    1: "EDDXXMDH",
    2: "E" + "D" * 32 + "H",
    3: "E" + "F" * 3 + "X" * 58 + "H",
    4: cfg4_pattern(),
    5: cfg5_pattern(),
}

CAP_180GB = 180 * 10**9


def config(cid: int, *, cap: Optional[int] = None) -> tuple:
    """(Problem, Space) of BASELINE.json configs[cid-1]."""
    tab = table_from_kinds(PATTERNS[cid], 1000 + cid)
    if cid == 1:
        pr = Problem(**tab, p=2, m=4, cap=INT64_MAX if cap is None else cap, name="cfg1")
        sp = Space([Group(1, FULL, combo_mask=0xF), Group(2, FULL), Group(4, FULL)])
    elif cid == 2:
        pr = Problem(**tab, p=4, m=16, cap=CAP_180GB if cap is None else cap, name="cfg2")
        sp = Space([Group(2, FULL, combo_mask=1 << ONEF1B)])
    elif cid == 3:
        pr = Problem(**tab, p=8, m=32, cap=CAP_180GB if cap is None else cap, name="cfg3")
        sp = Space([Group(1, BALL, 16, combo_mask=0xF), Group(2, BALL, 8, combo_mask=0x3F)])
    elif cid == 4:
        pr = Problem(**tab, p=8, m=64, cap=CAP_180GB if cap is None else cap, name="cfg4")
        sp = Space([Group(2, BALL, 8, combo_mask=0x3F)])
    elif cid == 5:
        pr = Problem(**tab, p=16, m=128, cap=CAP_180GB if cap is None else cap, name="cfg5")
        sp = Space([Group(1, BALL, 9, combo_mask=0xF), Group(2, BALL, 6, combo_mask=0x3F),
                    Group(4, BALL, 4, combo_mask=0x3F)])
    else:
        raise ValueError(cid)
    return pr, sp


def cfg1_unit() -> Problem:
    """SURVEY §8(c) hand-checkable unit instance of cfg1 (cap = infinity)."""
    t_f = [1, 4, 4, 6, 6, 3, 4, 5]
    t_w = [2, 4, 4, 6, 6, 2, 4, 6]
    z = [0] * 8
    return Problem(t_f=t_f, t_b=list(t_f), t_w=t_w, act=z, stash=z, weight=z, grad=z,
                   comm=[1] * 7 + [0], p=2, m=4, name="cfg1-unit")


def fractional_costs(pr: "Problem", rng: SplitMix64, denom: int = 8) -> np.ndarray:
    """[4][L] fp32 costs for the fp32 variant: each tick value plus a seeded
    fraction k/denom (durations stay >= 1)."""
    out = np.zeros((4, pr.L), np.float32)
    for ci, col in enumerate((pr.t_f, pr.t_b, pr.t_w, pr.comm)):
        for l in range(pr.L):
            out[ci, l] = np.float32(float(col[l]) + (rng.next() % denom) / denom)
    out[3, pr.L - 1] = 0.0
    return out


def random_problem(rng: SplitMix64, L: int, p: int, m: int, *, tmax: int = 9,
                   cmax: int = 4, bytes_max: int = 5, cap: int = INT64_MAX) -> Problem:
    """Small random heterogeneous tables for property tests."""
    def col(lo, hi):
        return [lo + int(rng.next() % (hi - lo + 1)) for _ in range(L)]
    return Problem(t_f=col(1, tmax), t_b=col(1, tmax), t_w=col(1, tmax),
                   act=col(0, bytes_max), stash=col(0, bytes_max), weight=col(0, bytes_max),
                   grad=col(0, bytes_max), comm=col(0, cmax), p=p, m=m, cap=cap)
