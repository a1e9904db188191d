"""The static-order kernel's host-built task order (adaptis_static_order, the
order `csrc/adaptis_fixed.cu` evaluates for GPIPE / ONEF1B / ZB segments),
checked on the CPU against the oracle's own fixed lists (readings R9-R11,
`oracle.fixed_order`) and by brute-force replay of its arrival slots:
  - restricted to one device, the order is that device's R9-R11 list
    (kind, stage and micro-batch, entry by entry);
  - every consumed slot holds exactly the item the entry consumes (F(s-1, j)
    for F(s, j), B(s+1, j) for B(s, j)), no slot is overwritten before it is
    consumed, and every produced item is consumed: the order is topological
    over the DAG edges, so max(free, arrival) + duration evaluated in it is the
    longest path of Lemma 1 for any durations;
  - the slot count is the number of slots used, and WAVE x ONEF1B (which R12
    excludes because Megatron's order deadlocks there) has no order."""
import pytest

from oracle import oracle as O
from paper_2509_23722_b200 import adaptis as A
from paper_2509_23722_b200 import workloads as W

CASES = [(pol, plc, p, v, m)
         for pol in (W.GPIPE, W.ONEF1B, W.ZB)
         for (plc, v) in ((W.SEQ, 1), (W.INTERLEAVED, 2), (W.INTERLEAVED, 4), (W.WAVE, 2), (W.WAVE, 3))
         for p in (1, 2, 3, 4, 5, 8)
         for m in ((1, 3, 7, 8, 16) if v == 1 else (p, 2 * p, 4 * p))
         if not (plc == W.WAVE and pol != W.GPIPE) and p * v <= 64]


def _oracle_lists(pol, plc, p, v, m):
    S = p * v
    pr = W.random_problem(W.SplitMix64(7), S + 1, p, m)
    cuts = list(range(S)) + [S + 1]
    return [[(k, s, j) for (k, s, j) in O.fixed_order(pr, v, plc, pol, cuts, d) if k in (0, 1)]
            for d in range(p)]


@pytest.mark.parametrize("pol,plc,p,v,m", CASES)
def test_static_order_is_the_lists_merged_topologically(pol, plc, p, v, m):
    ent, nslots = A.static_order(pol, plc, p, v, m)
    S = p * v
    assert len(ent) == 2 * S * m
    lists = _oracle_lists(pol, plc, p, v, m)
    pos = [0] * p
    nxt = {}                      # (kind, stage) -> next micro-batch in production order
    slot = {}                     # slot -> item held
    done = set()
    used = set()
    for (s, kind, ins, outs, d) in ent:
        j = nxt.get((kind, s), 0)
        nxt[(kind, s)] = j + 1
        # the device's list, entry by entry (R9-R11)
        assert pos[d] < len(lists[d]) and lists[d][pos[d]] == (kind, s, j), (d, pos[d], (kind, s, j))
        pos[d] += 1
        # the input: F(s-1, j) for F(s, j); B(s+1, j) for B(s, j); none at the ends
        want = ("F", s - 1, j) if kind == 0 and s > 0 else ("B", s + 1, j) if kind == 1 and s < S - 1 else None
        if want is None:
            assert ins is None
        else:
            assert ins is not None and slot.get(ins) == want, (ins, slot.get(ins), want)
            assert want in done
            del slot[ins]
        if kind == 1:
            assert ("F", s, j) in done  # its own F ran before (same device, earlier in the list)
        item = ("F" if kind == 0 else "B", s, j)
        has_out = s < S - 1 if kind == 0 else s > 0
        if has_out:
            assert outs is not None and outs not in slot, (outs, slot.get(outs))
            slot[outs] = item
            used.add(outs)
        else:
            assert outs is None
        done.add(item)
    assert pos == [len(lst) for lst in lists]
    assert not slot                # every produced item was consumed
    assert used == set(range(nslots))


def test_wave_onef1b_and_bad_arguments_have_no_order():
    with pytest.raises(A.AdaptisError):
        A.static_order(W.ONEF1B, W.WAVE, 4, 2, 8)   # R12: Megatron's order deadlocks on WAVE
    with pytest.raises(A.AdaptisError):
        A.static_order(W.GREEDY, W.INTERLEAVED, 4, 2, 8)
    with pytest.raises(A.AdaptisError):
        A.static_order(W.ONEF1B, W.INTERLEAVED, 4, 2, 6)  # R10 needs m % p == 0
    with pytest.raises(A.AdaptisError):
        A.static_order(W.ZB, W.INTERLEAVED, 32, 2, 32)    # p > 16: the lane kernels take it


def test_config_orders_fit_in_few_slots():
    """The configs' segments need at most 32 arrival slots."""
    for (pol, plc, p, v, m) in ((W.ONEF1B, W.INTERLEAVED, 8, 2, 32), (W.ZB, W.INTERLEAVED, 8, 2, 32),
                                (W.ONEF1B, W.INTERLEAVED, 4, 2, 16), (W.ZB, W.SEQ, 16, 1, 128),
                                (W.ONEF1B, W.INTERLEAVED, 16, 4, 128), (W.GPIPE, W.WAVE, 16, 2, 128)):
        _, ns = A.static_order(pol, plc, p, v, m)
        assert 1 <= ns <= 32, (pol, plc, p, v, m, ns)
