"""warpsim cross-check plumbing, on CPU.

The reference's warp lockstep simulator (proj/src/simd_sim.cpp) is reached
through oracle/_ref; scripts/warpsim_crosscheck.py compares its
memory_transactions with the sectors the device's thread-per-example Hogwild
kernel moves (ncu; profiles/round2_warpsim_crosscheck.jsonl). Here: the
wrapper reproduces the reference's own count_transactions known answers
(proj/tests/test_simd_sim.cpp:123-135, acceptance.cpp:379), and the per-kind
address streams the cross-check builds (data, model, writes with circular
offsets) add up to the simulator's total on the cross-check's datasets."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))


def test_count_transactions_known_answers(ref):
    assert ref.count_transactions([[0], [1], [2], [3]], 4) == 1
    assert ref.count_transactions([[0], [8], [16], [24]], 8) == 4
    assert ref.count_transactions([[l] for l in range(32)], 8) == 4


@pytest.mark.parametrize("layout,access", [("row-major", "row-rr"), ("row-major", "row-ch"),
                                           ("col-major", "col-rr"), ("col-major", "col-ch")])
def test_kind_split_reproduces_the_simulator(ref, layout, access):
    import warpsim_crosscheck as X
    host = ref.fixture_dense(X.N, X.D, X.SEED)
    ds = ref.convert_layout(host, 1) if layout == "col-major" else host
    _, st = ref.warpsim_epoch(ds, 0, 0.01, f"{access}:kernel:0", X.W, X.SEG, True)
    data, model, write, _ = X._streams(None, access, ref.assign(X.N, X.W, access.endswith("rr"), 0))
    split = sum(ref.count_transactions(v, X.SEG) for v in (data, model, write))
    assert split == st["memory_transactions"]
    assert st["surviving_updates"] <= st["attempted_updates"]
