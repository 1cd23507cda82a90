"""Randomised sweep of the integer host path against the unmodified reference's own Python module
(`oracle/_ref/_seqpar*.so`, compiled from /root/reference by oracle/Makefile; present in the
build container only, so the module is skipped elsewhere): layouts (naive / zigzag / usp,
partition.cpp:37-111), position ids and causal pair counts (:118-122, :160-162), pad_length
(:179-200), pick_xtuner_insp (attention.cpp:354-366) and the byte models (report.cpp:906-941),
bit-exact, including the inputs both sides reject."""
import os
import random
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
R = pytest.importorskip("_seqpar", reason="reference module not built (oracle/Makefile, build container only)")

import paper_2505_22296_b200 as P  # noqa: E402


def outcome(f, *a):
    """(value, None) or (None, 'error') — both sides raise ValueError subclasses on bad input."""
    try:
        return f(*a), None
    except ValueError:
        return None, "error"


def layout_cases(rng, n):
    out = []
    for _ in range(n):
        sp = rng.choice([1, 2, 3, 4, 6, 8, 16])
        mode = rng.choice(["naive", "zigzag", "usp"])
        u = r = 0
        if mode == "usp":
            divs = [d for d in range(1, sp + 1) if sp % d == 0]
            u = rng.choice(divs)
            r = sp // u
        L = rng.choice([rng.randrange(1, 300), 2 * sp * rng.randrange(1, 40), sp * rng.randrange(1, 64)])
        out.append((mode, L, sp, u, r))
    return out


def test_layouts_positions_pairs_match_reference():
    rng = random.Random(20261017)
    checked = 0
    for mode, L, sp, u, r in layout_cases(rng, 400):
        for i in range(sp):
            for name in ("shard_positions", "position_ids", "causal_pairs"):
                mine = outcome(getattr(P, name), mode, L, sp, i, u, r)
                ref = outcome(getattr(R, name), mode, L, sp, i, u, r)
                assert mine == ref, (name, mode, L, sp, i, u, r, mine, ref)
                checked += 1
    assert checked > 1000


def test_pad_length_matches_reference():
    rng = random.Random(7)
    for _ in range(3000):
        n = rng.choice([0, 1, rng.randrange(0, 5000), rng.randrange(0, 1 << 20)])
        sp = rng.choice([-1, 0, 1, 2, 3, 4, 8, 16])
        cutoff = rng.choice([0, 64, rng.randrange(0, 6000), 1 << 20])
        flag = rng.random() < 0.5
        assert outcome(P.pad_length, n, sp, cutoff, flag) == outcome(R.pad_length, n, sp, cutoff, flag), \
            (n, sp, cutoff, flag)


def test_xtuner_insp_matches_reference():
    rng = random.Random(11)
    for _ in range(2000):
        h = rng.randrange(1, 65)
        sp = rng.choice([1, 2, 3, 4, 6, 8, 12, 16])
        d = rng.choice([1, 2, 4, 8, 16, 24, 32, 48, 64, 96, 128])
        assert outcome(P.pick_xtuner_insp, h, sp, d) == outcome(R.pick_xtuner_insp, h, sp, d), (h, sp, d)


def test_byte_models_match_reference():
    rng = random.Random(13)
    for _ in range(1500):
        bs = rng.randrange(1, 4)
        sp = rng.choice([1, 2, 4, 8])
        L = 2 * sp * rng.randrange(1, 64)
        h = rng.randrange(1, 40)
        d = rng.choice([4, 8, 16, 64, 128])
        for name in ("ulysses_bytes", "ring_bytes", "dummy_head_bytes", "xtuner_bytes"):
            a = (bs, L, h, d, sp)
            assert outcome(getattr(P, name), *a) == outcome(getattr(R, name), *a), (name, a)
        u = rng.choice([d for d in range(1, sp + 1) if sp % d == 0])
        a = (bs, L, h, d, u, sp // u)
        assert outcome(P.usp_bytes, *a) == outcome(R.usp_bytes, *a), ("usp_bytes", a)
