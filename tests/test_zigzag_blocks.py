"""Block-wise zigzag layout (extension, no reference counterpart: ShardLayout::make_zigzag_blocks).
B = 1 must be the reference zigzag (pinned by the reference's own positions), B > 1 must match
the oracle restatement, and at config c5's document mix it must balance the ring's causal work
(busiest rank 19.5 % of the work under the single zigzag)."""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import seqpar_oracle as O  # noqa: E402

import paper_2505_22296_b200 as P  # noqa: E402

API = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_api.json")))["api"]


def test_one_block_is_the_reference_zigzag():
    for key, per_rank in API["positions"].items():
        mode, L, sp, u, r = key.split("/")
        if mode != "zigzag":
            continue
        L, sp = int(L), int(sp)
        for i in range(sp):
            assert P.shard_positions("zigzag:1", L, sp, i) == per_rank[i], key


@pytest.mark.parametrize("L,sp,B", [(64, 2, 2), (96, 4, 3), (256, 8, 2), (4096, 8, 16), (512, 1, 4)])
def test_blocks_match_oracle_and_partition(L, sp, B):
    owned = O.layout_owned(f"zigzag:{B}", L, sp)
    seen = []
    for i in range(sp):
        got = P.shard_positions(f"zigzag:{B}", L, sp, i)
        assert got == owned[i].tolist()
        assert len(got) == L // sp and got == sorted(got)
        assert P.causal_pairs(f"zigzag:{B}", L, sp, i) == int(np.sum(owned[i] + 1))
        seen += got
    assert sorted(seen) == list(range(L))


def test_bad_lengths_raise():
    with pytest.raises(ValueError):
        P.shard_positions("zigzag:3", 64, 2, 0)  # 64 % (2*2*3)
    with pytest.raises(ValueError):
        P.shard_positions("zigzag:0", 64, 2, 0)
    with pytest.raises(ValueError):
        P.shard_positions("zigzag:x", 64, 2, 0)


def test_c5_ring_balance():
    from sp_projection import c5_docs

    docs = c5_docs()
    L, sp = sum(docs), 8
    start = np.concatenate([[0], np.cumsum(docs)[:-1]])
    doc_of = np.repeat(np.arange(len(docs)), docs)
    work = np.arange(L) - start[doc_of] + 1  # keys each query admits within its document

    def busiest(mode):
        return max(work[np.array(P.shard_positions(mode, L, sp, i))].sum() for i in range(sp)) / work.sum()

    assert busiest("zigzag") > 0.19
    assert busiest("zigzag:16") < 0.13


def test_balanced_layout_choice():
    from sp_projection import c5_docs

    assert P.balanced_zigzag_layout(c5_docs(), 8) == "zigzag:16"
    # one document: the causal triangle of the whole sequence, which the single zigzag balances
    assert P.balanced_zigzag_layout([4096], 8) == "zigzag:1"
    # equal documents of whole chunks: the single zigzag is balanced already
    assert P.balanced_zigzag_layout([1024] * 8, 4) == "zigzag:1"
    # unequal documents: ranks 2 and 3 would carry 4x the work of ranks 0 and 1
    assert P.balanced_zigzag_layout([12288, 4096], 4, min_chunk=64) != "zigzag:1"
    with pytest.raises(ValueError):
        P.balanced_zigzag_layout([100], 8)
