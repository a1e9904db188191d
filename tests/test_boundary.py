"""The C-ABI boundary without a GPU: libadaptis.so loads, exports every entry
point include/adaptis.h declares, validates inputs naming the field, and its
host-side canonical order (adaptis_space_size / adaptis_decode, shared with
the kernels' decode) agrees with the oracle's independent recursive
enumerator and recursive-descent decoder."""
import ctypes as C
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2509_23722_b200 import adaptis as A
from paper_2509_23722_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(A.LIB_PATH)
    syms = A.exported_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s


def test_status_strings():
    lib = A.lib()
    assert lib.adaptis_status_str(0) == b"ok"
    assert lib.adaptis_status_str(2) == b"no feasible candidate"


def _small_spaces():
    rng = W.SplitMix64(8)
    for trial in range(10):
        p = 1 + rng.next() % 4
        m = p * (1 + rng.next() % 3)
        L = 4 * p + 2 + rng.next() % 5
        pr = W.random_problem(rng, L, p, m)
        groups = [W.Group(1, W.FULL, combo_mask=0xF)]
        if 2 * p <= L:
            groups.append(W.Group(2, W.BALL, 1 + rng.next() % 3, combo_mask=0x3F))
        if 3 * p <= L and trial % 2:
            groups.append(W.Group(3, W.BALL, 2, seed_cuts=list(range(1, 3 * p)), combo_mask=0x21))
        yield pr, W.Space(groups)


def test_space_size_and_decode_match_oracle_enumeration():
    for pr, sp in _small_spaces():
        n = A.space_size(pr, sp)
        assert n == O.space_size(pr, sp)
        for idx, plan in O.enumerate_space(pr, sp):
            assert A.decode(pr, sp, idx) == plan


def test_cfg1_cfg2_decode_exhaustive_sample():
    for cid in (1, 2):
        pr, sp = W.config(cid)
        N = A.space_size(pr, sp)
        assert N == O.space_size(pr, sp)
        idx = list(range(min(N, 3000))) + list(range(max(0, N - 500), N))
        want = dict(O.enumerate_space(pr, sp, limit=3000))
        for i in idx:
            got = A.decode(pr, sp, i)
            if i in want:
                assert got == want[i]
            assert got == O.decode(pr, sp, i)


@pytest.mark.parametrize("cid", [3, 4, 5])
def test_ball_configs_decode_matches_oracle_random_access(cid):
    """BALL spaces: the library's closed-form counts + seed vs the oracle's
    recursive counts + DP seed, on 400 seeded indices per config."""
    pr, sp = W.config(cid)
    N = A.space_size(pr, sp)
    assert N == O.space_size(pr, sp)
    rng = np.random.default_rng(12345)
    for i in list(rng.integers(0, N, 400)) + [0, N - 1]:
        assert A.decode(pr, sp, int(i)) == O.decode(pr, sp, int(i))


def test_validation_names_the_field():
    pr, sp = W.config(1)
    bad = W.Problem(**{c: getattr(pr, c).copy() for c in W.COLUMNS}, p=pr.p, m=pr.m)
    bad.t_f[3] = 0
    with pytest.raises(A.AdaptisError, match=r"layers\.t_f\[3\] < 1"):
        A.space_size(bad, sp)
    bad2 = W.Problem(**{c: getattr(pr, c).copy() for c in W.COLUMNS}, p=pr.p, m=3)
    with pytest.raises(A.AdaptisError, match=r"m % p == 0"):
        A.space_size(bad2, sp)
    with pytest.raises(A.AdaptisError, match="combo_mask"):
        A.space_size(pr, W.Space([W.Group(1, W.FULL, combo_mask=0x10)]))
    with pytest.raises(A.AdaptisError, match="index"):
        A.decode(pr, sp, 244)


def test_overflow_is_reported():
    pr = W.Problem(t_f=[1 << 52] * 8, t_b=[1] * 8, t_w=[1] * 8, act=[0] * 8, stash=[0] * 8,
                   weight=[0] * 8, grad=[0] * 8, comm=[0] * 8, p=2, m=64)
    with pytest.raises(A.AdaptisError) as e:
        A.space_size(pr, W.Space([W.Group(1, W.FULL, combo_mask=0xF)]))
    assert e.value.status == A.EOVERFLOW


def test_ctypes_layouts_match_header(tmp_path):
    """The binding's ctypes structures have the sizes and field offsets the C
    compiler gives the structs of include/adaptis.h (ABI check, no GPU)."""
    import ctypes as C
    import subprocess
    from paper_2509_23722_b200 import adaptis as A
    src = tmp_path / "layout.c"
    src.write_text(r'''
#include <stddef.h>
#include <stdio.h>
#include "adaptis.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(adaptis_problem), sizeof(adaptis_plan),
         sizeof(adaptis_result), sizeof(adaptis_best), offsetof(adaptis_best, comm_d),
         offsetof(adaptis_best, n_candidates), sizeof(adaptis_gen_result),
         offsetof(adaptis_gen_result, step_makespan), sizeof(adaptis_launch_info),
         sizeof(adaptis_gen_options));
  return 0;
}
''')
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    want = [C.sizeof(A._Problem), C.sizeof(A._Plan), C.sizeof(A._Result), C.sizeof(A._Best),
            A._Best.comm_d.offset, A._Best.n_candidates.offset, C.sizeof(A._GenResult),
            A._GenResult.step_makespan.offset, C.sizeof(A._LaunchInfo), C.sizeof(A._GenOptions)]
    assert got == want
