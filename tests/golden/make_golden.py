"""Regenerates the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Runs only in the build container (needs /root/reference and `make -C oracle ref`):
  * ``oracle/_ref/ref_driver`` (our driver over the reference library) for attention values
    and gradients (single device) and for sharded engine runs with per-rank byte counters;
  * the reference's own pybind module ``oracle/_ref/_seqpar`` for layouts, padding, xtuner
    factors and the closed-form byte models.
The fixtures are committed; tests never need /root/reference at run time.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = os.path.join(ROOT, "oracle", "_ref")
DRIVER = os.path.join(REF, "ref_driver")


def read_arrays(path):
    out = []
    with open(path, "rb") as f:
        while True:
            hdr = f.read(8)
            if not hdr:
                break
            n = int(np.frombuffer(hdr, np.int64)[0])
            out.append(np.frombuffer(f.read(8 * n), np.float64).copy())
    return out


ATTN_CASES = [
    # name, L, heads, kv, dim, causal, seed
    ("attn_L32_h4_d8", 32, 4, 4, 8, 1, 7),
    ("attn_L64_h6_kv2_d8", 64, 6, 2, 8, 1, 11),
    ("attn_L48_h2_kv1_d16_bidir", 48, 2, 1, 16, 0, 3),
    ("attn_L40_h3_d4", 40, 3, 3, 4, 1, 1000003 + 5),
]

ENGINE_CASES = [
    # engine, sp, L, heads, kv, dim, u, r, seed
    ("ulysses", 2, 32, 4, 4, 8, 0, 0, 1000003),
    ("ulysses", 4, 64, 8, 2, 8, 0, 0, 1000004),
    ("dummy_head", 4, 32, 6, 6, 8, 0, 0, 1000005),
    ("dummy_head", 8, 32, 14, 2, 4, 0, 0, 1000006),
    ("xtuner", 4, 32, 6, 6, 8, 0, 0, 1000007),
    ("ring", 2, 32, 4, 4, 8, 0, 0, 1000008),
    ("ring", 4, 64, 4, 2, 8, 0, 0, 1000009),
    ("ring", 8, 64, 2, 2, 4, 0, 0, 1000010),
    ("usp", 4, 64, 4, 4, 8, 2, 2, 1000011),
]


ROPE_CASES = [
    # name, L, heads, dim, pos_scale, pos_offset, seed
    ("rope_L16_h2_d8", 16, 2, 8, 1, 0, 13),
    ("rope_L12_h3_d6_far", 12, 3, 6, 7, 100000, 17),
    ("rope_L8_h2_d64_far", 8, 2, 64, 1000, 3, 19),
    ("rope_L6_h1_d16_neg", 6, 1, 16, -5, 2, 23),
]

ROPE_ENGINE_CASES = [
    # engine, sp, L, heads, kv, dim, u, r, pos_scale, pos_offset, seed
    ("ulysses", 2, 32, 4, 2, 8, 0, 0, 1, 0, 2000001),
    ("ulysses", 4, 64, 8, 2, 16, 0, 0, 3, 5000, 2000002),
    ("dummy_head", 4, 32, 6, 2, 8, 0, 0, 1, 0, 2000003),
    ("xtuner", 4, 32, 6, 6, 8, 0, 0, 1, 0, 2000004),
    ("ring", 4, 64, 4, 2, 8, 0, 0, 1, 0, 2000005),
    ("usp", 4, 64, 4, 4, 8, 2, 2, 1, 0, 2000006),
    ("oracle", 1, 32, 4, 2, 8, 0, 0, 1, 7, 2000007),
]


def make_rope(tmp):
    """rope_apply (tensor.cpp:548-607) alone, and the engines with q/k rotated at global ids
    (Model::forward, model.cpp:339-344) -> tests/golden/reference_rope.npz."""
    arrays = {}
    for name, L, h, d, sc, off, seed in ROPE_CASES:
        p = os.path.join(tmp, name + ".bin")
        subprocess.run([DRIVER, "rope", str(L), str(h), str(d), str(sc), str(off), str(seed), p],
                       check=True)
        x, R, y, dx = read_arrays(p)
        for key, val in dict(x=x, R=R, y=y, dx=dx).items():
            arrays[f"{name}/{key}"] = val
        arrays[f"{name}/meta"] = np.array([L, h, d, sc, off, seed], np.int64)
    for eng, sp, L, h, kv, d, u, r, sc, off, seed in ROPE_ENGINE_CASES:
        name = f"rope_engine_{eng}_sp{sp}_L{L}_h{h}_kv{kv}_d{d}"
        p = os.path.join(tmp, name + ".bin")
        subprocess.run([DRIVER, "rope_engine", eng, str(sp), str(L), str(h), str(kv), str(d),
                        str(u), str(r), str(sc), str(off), str(seed), p], check=True)
        out, dq, dk, dv, tot, a2a, ag, p2p = read_arrays(p)
        for key, val in dict(out=out, dq=dq, dk=dk, dv=dv).items():
            arrays[f"{name}/{key}"] = val
        arrays[f"{name}/meta"] = np.array([sp, L, h, kv, d, u, r, sc, off, seed], np.int64)
        arrays[f"{name}/engine"] = np.frombuffer(eng.encode().ljust(16, b" "), np.uint8)
    np.savez_compressed(os.path.join(HERE, "reference_rope.npz"), **arrays)
    print("wrote", os.path.join(HERE, "reference_rope.npz"))


BATCH_CASES = [
    # len, sp, cutoff_len, pad_to_cutoff, seed
    (13, 2, 512, 0, 3), (37, 4, 1024, 0, 5), (50, 2, 256, 1, 7), (64, 8, 64, 0, 11),
    (5, 1, 64, 0, 13), (100, 4, 128, 1, 17),
]


def make_batch():
    """pad_batch / split_position_map / replicate_packing_mask of the unmodified reference ->
    tests/golden/reference_batch.json."""
    out = []
    for ln, sp, cut, to_cut, seed in BATCH_CASES:
        r = subprocess.run([DRIVER, "batch", str(ln), str(sp), str(cut), str(to_cut), str(seed)],
                           check=True, capture_output=True, text=True)
        rec = json.loads(r.stdout)
        rec["args"] = [ln, sp, cut, to_cut, seed]
        out.append(rec)
    with open(os.path.join(HERE, "reference_batch.json"), "w") as f:
        json.dump(out, f)
    print("wrote", os.path.join(HERE, "reference_batch.json"))


def make_loss():
    """sequence_logprob_per_position / sft_loss_sharded / dpo_loss_sharded of the unmodified
    reference on its own test inputs -> tests/golden/reference_loss.json."""
    r = subprocess.run([DRIVER, "loss"], check=True, capture_output=True, text=True)
    with open(os.path.join(HERE, "reference_loss.json"), "w") as f:
        f.write(r.stdout)
    print("wrote", os.path.join(HERE, "reference_loss.json"))


def main():
    if not os.path.exists(DRIVER):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    tmp = tempfile.mkdtemp()
    arrays = {}
    for name, L, h, kv, d, causal, seed in ATTN_CASES:
        p = os.path.join(tmp, name + ".bin")
        subprocess.run([DRIVER, "golden", str(L), str(h), str(kv), str(d), str(causal),
                        str(seed), p], check=True)
        q, k, v, R, out, lse, dq, dk, dv = read_arrays(p)
        for key, val in dict(q=q, k=k, v=v, R=R, out=out, lse=lse, dq=dq, dk=dk, dv=dv).items():
            arrays[f"{name}/{key}"] = val
        arrays[f"{name}/meta"] = np.array([L, h, kv, d, causal, seed], np.int64)
    for eng, sp, L, h, kv, d, u, r, seed in ENGINE_CASES:
        name = f"engine_{eng}_sp{sp}_L{L}_h{h}_kv{kv}_d{d}"
        p = os.path.join(tmp, name + ".bin")
        subprocess.run([DRIVER, "engine", eng, str(sp), str(L), str(h), str(kv), str(d), str(u),
                        str(r), str(seed), p], check=True)
        out, dq, dk, dv, tot, a2a, ag, p2p = read_arrays(p)
        for key, val in dict(out=out, dq=dq, dk=dk, dv=dv, bytes=tot, a2a_bytes=a2a,
                             all_gather_bytes=ag, p2p_bytes=p2p).items():
            arrays[f"{name}/{key}"] = val
        arrays[f"{name}/meta"] = np.array([sp, L, h, kv, d, u, r, seed], np.int64)
        arrays[f"{name}/engine"] = np.frombuffer(eng.encode().ljust(16, b" "), np.uint8)
    np.savez_compressed(os.path.join(HERE, "reference_attention.npz"), **arrays)

    # full-size config 1 (L=4096, 8 heads, d=64, causal): checksums only (the arrays are 16 MB)
    p = os.path.join(tmp, "c1.bin")
    subprocess.run([DRIVER, "golden", "4096", "8", "8", "64", "1", "1", p], check=True)
    q, k, v, R, out, lse, dq, dk, dv = read_arrays(p)
    c1 = {}
    for key, val in dict(q=q, out=out, lse=lse, dq=dq, dk=dk, dv=dv).items():
        shaped = val.reshape(4096, 8, -1) if key != "lse" else val.reshape(4096, 8, 1)
        c1[key] = {"sum_per_head": shaped.sum(axis=(0, 2)).tolist(),
                   "abs_sum": float(np.abs(val).sum()),
                   "rows_0_1_4095": shaped[[0, 1, 4095]].tolist()}
    c1["meta"] = {"L": 4096, "heads": 8, "kv": 8, "dim": 64, "causal": 1, "seed": 1}

    # layouts, padding, byte models straight from the reference's Python API
    sys.path.insert(0, REF)
    import _seqpar as S  # noqa: E402

    api = {"positions": {}, "causal_pairs": {}, "pad_length": [], "insp": [], "bytes": [],
           "measured_bytes": []}
    for mode, L, sp, u, r in [("naive", 8, 2, 0, 0), ("zigzag", 8, 2, 0, 0),
                              ("zigzag", 32, 4, 0, 0), ("zigzag", 64, 8, 0, 0),
                              ("usp", 32, 4, 2, 2), ("usp", 64, 8, 2, 4), ("usp", 64, 8, 4, 2),
                              ("naive", 48, 3, 0, 0)]:
        key = f"{mode}/{L}/{sp}/{u}/{r}"
        api["positions"][key] = [S.shard_positions(mode, L, sp, i, u, r) for i in range(sp)]
        api["causal_pairs"][key] = [S.causal_pairs(mode, L, sp, i, u, r) for i in range(sp)]
    for args in [(13, 2, 512, False), (16, 2, 512, False), (13, 4, 512, False),
                 (50, 2, 1024, False), (50, 1, 1024, False), (64, 2, 64, False),
                 (5, 4, 256, False), (50, 2, 256, True), (262144, 8, 262144, False)]:
        api["pad_length"].append([*args, S.pad_length(*args)])
    for args in [(6, 4, 8), (14, 8, 4), (28, 8, 128), (7, 8, 64), (32, 8, 128), (6, 4, 64)]:
        api["insp"].append([*args, S.pick_xtuner_insp(*args)])
    for fn, args in [("ulysses_bytes", (1, 64, 4, 8, 4)), ("ring_bytes", (1, 32, 2, 4, 4)),
                     ("dummy_head_bytes", (1, 32, 14, 4, 8)),
                     ("xtuner_bytes", (1, 32, 14, 4, 8)), ("usp_bytes", (1, 64, 4, 8, 4, 1)),
                     ("usp_bytes", (1, 64, 4, 8, 2, 2)), ("usp_bytes", (1, 64, 4, 8, 1, 4)),
                     ("ulysses_bytes", (1, 4096, 8, 64, 2)),
                     ("dummy_head_bytes", (1, 65536, 28, 128, 8)),
                     ("xtuner_bytes", (1, 65536, 28, 128, 8)),
                     ("ring_bytes", (1, 131072, 32, 128, 8))]:
        api["bytes"].append([fn, list(args), getattr(S, fn)(*args)])
    for eng, L, h, kv, d, sp, u, r in [("ulysses", 64, 4, 4, 8, 4, 0, 0),
                                       ("ulysses", 64, 4, 2, 8, 4, 0, 0),
                                       ("ring", 32, 2, 2, 4, 4, 0, 0),
                                       ("dummy_head", 32, 14, 14, 4, 8, 0, 0),
                                       ("xtuner", 32, 14, 14, 4, 8, 0, 0),
                                       ("usp", 64, 4, 4, 8, 4, 2, 2)]:
        api["measured_bytes"].append([eng, L, h, kv, d, sp, u, r,
                                      S.measure_engine_bytes(eng, L, h, kv, d, sp, u, r)])
    with open(os.path.join(HERE, "reference_api.json"), "w") as f:
        json.dump({"api": api, "c1": c1}, f, indent=1)
    print("wrote", os.path.join(HERE, "reference_attention.npz"), "and reference_api.json")


if __name__ == "__main__":
    if sys.argv[1:] == ["rope"]:
        make_rope(tempfile.mkdtemp())
    elif sys.argv[1:] == ["batch"]:
        make_batch()
    elif sys.argv[1:] == ["loss"]:
        make_loss()
    else:
        main()
        make_rope(tempfile.mkdtemp())
        make_batch()
        make_loss()
