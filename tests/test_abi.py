"""CPU checks of the C-ABI boundary: libspattn.so loads without a GPU, exports every symbol
include/spattn.h declares, and its host (integer) functions reproduce the reference's golden
layouts, padding, xtuner factors and byte models (tests/golden/reference_api.json)."""
import ctypes
import json
import os
import re

import pytest

from paper_2505_22296_b200 import _lib as C
import paper_2505_22296_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
API = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_api.json")))["api"]


def header_symbols():
    text = open(os.path.join(ROOT, "include", "spattn.h")).read()
    return sorted(set(re.findall(r"\b(spattn_\w+)\s*\(", text)))


def test_header_and_binding_agree():
    assert header_symbols() == sorted(C.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = C.lib()
    for name in header_symbols():
        assert hasattr(L, name), name
    assert L.spattn_abi_version() == 1


def test_layout_positions_and_pairs_match_reference():
    for key, per_rank in API["positions"].items():
        mode, L, sp, u, r = key.split("/")
        L, sp, u, r = int(L), int(sp), int(u), int(r)
        for i in range(sp):
            assert P.shard_positions(mode, L, sp, i, u, r) == per_rank[i], key
            assert P.causal_pairs(mode, L, sp, i, u, r) == API["causal_pairs"][key][i], key


def test_pad_length_insp_bytes_match_reference():
    for *args, want in API["pad_length"]:
        assert P.pad_length(*args) == want
    for *args, want in API["insp"]:
        assert P.pick_xtuner_insp(*args) == want
    for fn, args, want in API["bytes"]:
        assert getattr(P, fn)(*args) == want, (fn, args)


def test_errors_map_to_value_error():
    # tests/test_partition.cpp:82-89 and attention.cpp:354-366 rejects
    with pytest.raises(ValueError):
        P.shard_positions("naive", 10, 4, 0)
    with pytest.raises(ValueError):
        P.shard_positions("zigzag", 12, 4, 0)
    with pytest.raises(ValueError):
        P.pick_xtuner_insp(3, 4, 9)
    with pytest.raises(ValueError):
        P.pad_length(50, 2, 32)
    with pytest.raises(ValueError):
        P.shard_positions("bogus", 16, 2, 0)
    msg = C.lib().spattn_last_error().decode()
    assert msg  # thread-local message of the last failing call


def test_binding_arity_matches_header():
    """Every ctypes binding declares as many arguments as the C prototype has parameters."""
    text = re.sub(r"/\*.*?\*/", "", open(os.path.join(ROOT, "include", "spattn.h")).read(), flags=re.S)
    L = C.lib()
    for m in re.finditer(r"\b(spattn_\w+)\s*\(([^)]*)\)\s*;", text):
        name, params = m.group(1), m.group(2).strip()
        n = 0 if params in ("", "void") else params.count(",") + 1
        at = getattr(L, name).argtypes
        assert at is None or len(at) == n, (name, n, len(at))


def test_header_is_plain_c_and_links(tmp_path):
    """The boundary is a C ABI: a plain C program (gcc, no C++) includes spattn.h, links
    libspattn.so and calls the host-side entry points (what a cgo / JNI / FFI stub does)."""
    import shutil
    import subprocess

    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    src = tmp_path / "abi.c"
    src.write_text(r'''
#include <stdio.h>
#include "spattn.h"
int main(void) {
  int64_t n = 0, pairs = 0;
  if (spattn_abi_version() != 1) return 1;
  if (spattn_pad_length(1000, 4, 2048, 0, &n) != 0) return 2;
  spattn_layout lay = {0};
  lay.mode = 1; lay.sp = 2; lay.global_len = 8;  /* zigzag(8, 2) */
  int64_t pos[4];
  if (spattn_layout_positions(&lay, 0, pos) != 0) return 3;
  if (spattn_causal_pairs(&lay, 0, &pairs) != 0) return 4;
  if (spattn_pad_length(10, 4, 3, 0, &n) == 0) return 5;  /* cutoff below len*: an error code */
  printf("%lld %lld %lld %lld %lld %s\n", (long long)pos[0], (long long)pos[1], (long long)pos[2],
         (long long)pos[3], (long long)pairs, spattn_last_error());
  return 0;
}
''')
    exe = tmp_path / "abi"
    libdir = os.path.dirname(C.LIB_PATH)
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), str(src),
                    "-L", libdir, "-l:" + os.path.basename(C.LIB_PATH), "-Wl,-rpath," + libdir, "-o", str(exe)],
                   check=True, capture_output=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, (out.returncode, out.stderr)
    vals = out.stdout.split()
    assert [int(x) for x in vals[:5]] == [0, 1, 6, 7, 18]  # tests/test_partition.cpp:19-33
