"""Batches, padding to 8*sp and neat-packing metadata (reference partition.hpp:92-125,
partition.cpp:164-227): the oracle and the C-ABI host functions against fixtures from the
unmodified reference (tests/golden/reference_batch.json), the reference's own cases
(tests/test_partition.cpp:151-235), and on the GPU the packing-mask broadcast and the packed
batch driving the varlen kernels with per-document rope ids."""
import json
import os

import numpy as np
import pytest

import seqpar_oracle as O
import paper_2505_22296_b200 as P

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_batch.json")))


@pytest.mark.parametrize("rec", GOLD, ids=[str(r["args"]) for r in GOLD])
def test_pad_batch_matches_reference(rec):
    ln, sp, cut, to_cut, _ = rec["args"]
    b = P.TrainBatch(rec["tokens"], rec["labels"], list(range(ln)), rec["segment_ids"],
                     rec["image_map"])
    p = P.pad_batch(b, sp, 7, cut, bool(to_cut))
    want = (rec["p_tokens"], rec["p_labels"], rec["p_position_ids"], rec["p_segment_ids"],
            rec["p_image_map"])
    assert (p.tokens, p.labels, p.position_ids, p.segment_ids, p.image_map) == want
    assert O.pad_batch(rec["tokens"], rec["labels"], list(range(ln)), rec["segment_ids"],
                       rec["image_map"], sp, 7, cut, bool(to_cut)) == want
    for i in range(sp):
        assert P.split_position_map(p.image_map, "zigzag", sp, i) == rec["split_image_map"][i]
    # the varlen bridge agrees with the oracle's restatement
    assert P.documents_from_segments(p.segment_ids) == O.documents_from_segments(p.segment_ids)
    assert sum(P.documents_from_segments(p.segment_ids)) == len(p)


def test_pad_batch_sentinels():
    # tests/test_partition.cpp:151-176
    b = P.TrainBatch([5, 6, 7], [5, P.IGNORE_LABEL, 7], [0, 1, 2], [0, 0, 1], [P.NO_IMAGE, 3, P.NO_IMAGE])
    p = P.pad_batch(b, 1, 0, 64)
    assert len(p) == 8 and p.tokens == [5, 6, 7, 0, 0, 0, 0, 0]
    assert p.labels[3] == P.IGNORE_LABEL and p.labels[7] == P.IGNORE_LABEL
    assert p.position_ids == list(range(8))
    assert p.segment_ids == [0, 0, 1] + [P.NO_SEGMENT] * 5
    assert p.image_map[4] == P.NO_IMAGE
    p.validate()
    p2 = P.pad_batch(P.TrainBatch([1, 2], [1, 2], [0, 1]), 2, 0, 128)
    assert len(p2) == 16 and p2.segment_ids == [] and p2.image_map == []


def test_padded_batches_shard_cleanly():
    # tests/test_partition.cpp:178-191
    p = P.pad_batch(P.TrainBatch([9] * 37, [9] * 37, list(range(37))), 4, 0, 1024)
    assert len(p) == 64
    for i in range(4):
        assert len(P.split_position_map(p.tokens, "zigzag", 4, i)) == 16


def test_image_map_sharding_follows_layout():
    # tests/test_partition.cpp:193-202
    m = [P.NO_IMAGE] * 8
    m[2], m[3], m[6] = 0, 1, 2
    assert P.split_position_map(m, "zigzag", 2, 0) == [P.NO_IMAGE, P.NO_IMAGE, 2, P.NO_IMAGE]
    assert P.split_position_map(m, "zigzag", 2, 1) == [0, 1, P.NO_IMAGE, P.NO_IMAGE]


def test_batch_validation():
    # tests/test_partition.cpp:204-214
    b = P.TrainBatch([1, 2, 3], [1, 2], [0, 1, 2])
    with pytest.raises(P.ConfigError):
        b.validate()
    with pytest.raises(P.ConfigError):
        P.pad_batch(b, 1, 0, 64)
    b.labels = [1, 2, 3]
    b.validate()
    b.image_map = [0]
    with pytest.raises(P.ConfigError):
        b.validate()
    with pytest.raises(P.ConfigError):  # padded length beyond the cutoff (partition.cpp:195-197)
        P.pad_batch(P.TrainBatch([1] * 100, [1] * 100, list(range(100))), 4, 0, 64)


def test_documents_from_segments():
    assert P.documents_from_segments([0, 0, 1, 1, 1, -1, -1]) == [2, 3, 2]
    assert P.documents_from_segments([3]) == [1]
    with pytest.raises(P.ConfigError):
        P.documents_from_segments([0, 0, 1, 0])
    with pytest.raises(O.ConfigError):
        O.documents_from_segments([0, 0, 1, 0])
    assert P.document_position_ids([2, 3]) == [0, 1, 0, 1, 2]


# ---------------------------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("rec", GOLD, ids=[str(r["args"]) for r in GOLD])
def test_gpu_replicate_packing_mask_matches_reference(rec):
    sp = rec["args"][1]
    mask = bytes(rec["mask"])
    fab = P.Fabric(sp)
    fab.reset_stats()
    got = fab.replicate_packing_mask([mask] + [None] * (sp - 1))
    assert all(g == mask for g in got)
    assert [fab.stats(r)["broadcast"][1] for r in range(sp)] == rec["broadcast_bytes"]


@pytest.mark.gpu
@pytest.mark.parametrize("engine,sp", [("ulysses", 4), ("ring", 2), ("dummy_head", 4)])
def test_gpu_packed_batch_drives_varlen_attention(engine, sp):
    """Neat packing end to end: a packed batch is padded to 8*sp, its segment ids become the
    varlen documents and its per-document reset ids the rope positions; the sharded engine
    matches the composed per-document oracle (rope at reset ids, oracle_attention per doc)."""
    import torch
    from gpu_util import assert_close, np_, parity_inputs, to_dev, torch_ref

    P.set_kernel_family("tcgen05")
    rng = np.random.default_rng(sp)
    lens = [int(x) for x in rng.integers(20, 90, 4)]
    n = sum(lens)
    seg = [i for i, m in enumerate(lens) for _ in range(m)]
    b = P.pad_batch(P.TrainBatch(list(range(n)), list(range(n)), list(range(n)), seg), sp, 0, 4096)
    docs = P.documents_from_segments(b.segment_ids)
    ids = P.document_position_ids(docs)
    L, H, Hkv, d = len(b), 4, 2, 64
    q, k, v, R = parity_inputs(900 + sp, L, H, Hkv, d)
    qt, kt, vt = (to_dev(x).requires_grad_(True) for x in (q, k, v))
    out = P.engine_attention(engine, qt, kt, vt, sp, docs=docs, position_ids=ids)
    (out.float() * to_dev(R).float()).sum().backward()
    qr, kr = O.rope_apply(q, ids), O.rope_apply(k, ids)
    orc = O.varlen_attention_fwd_bwd(qr, kr, v, R, docs)
    orc["dq"] = O.rope_apply(orc["dq"], ids, inverse=True)
    orc["dk"] = O.rope_apply(orc["dk"], ids, inverse=True)
    ref = torch_ref(O.bf16_round(qr), O.bf16_round(kr), v, R, docs=docs)
    ref["dq"] = O.bf16_round(O.rope_apply(ref["dq"], ids, inverse=True))
    ref["dk"] = O.bf16_round(O.rope_apply(ref["dk"], ids, inverse=True))
    got = {"out": np_(out), "dq": np_(qt.grad), "dk": np_(kt.grad), "dv": np_(vt.grad)}
    for key in got:
        assert_close(key, got[key], orc[key], ref[key])
    torch.cuda.synchronize()
