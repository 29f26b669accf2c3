"""CPU checks of the C-ABI boundary: the library builds, loads, exports every
symbol include/kascade_b200.h declares, and rejects bad arguments with the
reference's error classes before any launch (no GPU needed)."""

import ctypes
import os
import re

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "kascade_b200.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2512_16391_b200 import _lib, build
    build.build()
    return _lib.load()


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int32_t|const char\*)\s+(kscd_\w+)\s*\(", text, re.M)))


def test_every_declared_symbol_is_exported(lib):
    names = declared_functions()
    assert len(names) >= 8
    for name in names:
        assert hasattr(lib, name), name


def test_abi_version_and_k_budget(lib):
    assert lib.kscd_abi_version() == 2
    # tiles.py:81-89 pins (pkg/tests/test_tiles.py:18-23)
    for n, k in ((64, 64), (1000, 128), (1280, 128), (4096, 409)):
        assert lib.kscd_k_budget(0.1, 128, n) == k
    assert lib.kscd_k_budget(0.1, 1, 4096) == 409  # floor, not round
    assert lib.kscd_k_budget(1.0, 4096, 10) == 10


def test_invalid_arguments_map_to_reference_errors(lib):
    from paper_2512_16391_b200 import _lib
    from paper_2512_16391_b200.exceptions import InvalidArgumentError, UnsupportedOperationError
    p = _lib.DecodeParams(batch=1, num_q_heads=8, num_kv_heads=2, head_dim=129, seq_len=4)
    with pytest.raises(UnsupportedOperationError):
        _lib.call("kscd_dense_decode", p, 0)
    p.head_dim = 0
    with pytest.raises(UnsupportedOperationError):
        _lib.call("kscd_dense_decode", p, 0)
    p.head_dim = 64                 # logical d < 128: rows zero-padded to 128 (header Conventions)
    p.num_kv_heads = 3
    with pytest.raises(InvalidArgumentError, match="divisible"):
        _lib.call("kscd_dense_decode", p, 0)
    p.num_kv_heads = 2
    with pytest.raises(InvalidArgumentError, match="non-NULL"):
        _lib.call("kscd_sparse_decode", p, 0)
    t = _lib.TopkParams(rows=1, values=1, length=5, k=0, indices=1, counts=1, k_cap=1)
    with pytest.raises(InvalidArgumentError, match="k must be >= 1"):
        _lib.call("kscd_topk", t, 0)
    s = _lib.SelectDecodeParams(batch=1, num_q_heads=8, num_kv_heads=2, seq_len=10, topk_fraction=0.0, k_min=1)
    with pytest.raises(InvalidArgumentError, match="fraction"):
        _lib.call("kscd_select_decode", s, 0)


def test_workspace_size_query(lib):
    from paper_2512_16391_b200 import _lib
    p = _lib.DecodeParams(batch=8, num_q_heads=32, num_kv_heads=8, head_dim=128, seq_len=131072)
    nb = ctypes.c_size_t(0)
    assert lib.kscd_decode_workspace_size(ctypes.byref(p), ctypes.byref(nb)) == 0
    assert nb.value >= 8 * 32 * 130 * 4


STRUCTS = {"kscd_decode_params": "DecodeParams", "kscd_select_decode_params": "SelectDecodeParams",
           "kscd_topk_params": "TopkParams", "kscd_prefill_params": "PrefillParams",
           "kscd_select_prefill_params": "SelectPrefillParams", "kscd_probs_params": "ProbsParams",
           "kscd_pool_tiles_params": "PoolTilesParams", "kscd_append_kv_params": "AppendKvParams",
           "kscd_masked_mass_params": "MaskedMassParams", "kscd_select_pre_params": "SelectPreParams",
           "kscd_decode_layers": "DecodeLayers"}


def _header_fields():
    """Member names of every params struct, in declaration order."""
    text = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    out = {}
    for name, body in re.findall(r"typedef struct (kscd_\w+)\s*\{(.*?)\}\s*\1\s*;", text, re.S):
        fields = []
        for decl in body.split(";"):
            decl = decl.strip()
            if not decl:
                continue
            head, *rest = decl.split(",")
            fields.append(re.findall(r"(\w+)\s*$", head)[0])
            fields.extend(r.strip().lstrip("*").strip() for r in rest)
        out[name] = fields
    return out


def test_ctypes_structs_match_the_header_layout(tmp_path):
    """Every params struct of the C ABI: the ctypes binding declares the same
    members in the same order at the same byte offsets, with the same size,
    as gcc lays out include/kascade_b200.h."""
    import shutil
    import subprocess
    from paper_2512_16391_b200 import _lib
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    fields = _header_fields()
    assert set(fields) == set(STRUCTS), sorted(fields)
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "kascade_b200.h"', "int main(void) {"]
    for cname, members in fields.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for m in members:
            lines.append(f'  printf("{cname} {m} %zu\\n", offsetof({cname}, {m}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(REPO, "include"), str(src), "-o", str(exe)], check=True)
    c_layout = {}
    for line in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        struct, member, value = line.split()
        c_layout[(struct, member)] = int(value)
    for cname, pyname in STRUCTS.items():
        cls = getattr(_lib, pyname)
        names = [f[0] for f in cls._fields_]
        assert names == fields[cname], (cname, names, fields[cname])
        assert ctypes.sizeof(cls) == c_layout[(cname, "size")], cname
        for m in names:
            assert getattr(cls, m).offset == c_layout[(cname, m)], (cname, m)


def test_workspace_covers_virtual_heads_of_large_groups(lib):
    """Query groups above 16 run as virtual kv heads (G = 32 -> 2 per kv
    head): the workspace query counts their split counters too."""
    from paper_2512_16391_b200 import _lib

    def size(hq, hkv):
        p = _lib.DecodeParams(batch=4, num_q_heads=hq, num_kv_heads=hkv, head_dim=128, seq_len=4096)
        nb = ctypes.c_size_t(0)
        assert lib.kscd_decode_workspace_size(ctypes.byref(p), ctypes.byref(nb)) == 0
        return nb.value

    # same query heads; one kv head with G = 32 needs counters for 2 virtual heads
    assert size(32, 1) >= 4 * 32 * 130 * 4 + 4 * 2 * 4
    assert size(32, 2) >= 4 * 32 * 130 * 4 + 4 * 2 * 4


def test_integration_stub_matches_header():
    """INTEGRATION.md's raw ctypes stub for kscd_decode_params lists every
    member of the header's struct, in order (a short stub would make the
    library read past the caller's struct)."""
    from paper_2512_16391_b200 import _lib
    text = open(os.path.join(REPO, "INTEGRATION.md")).read()
    body = text[text.index("class kscd_decode_params"):]
    body = body[:body.index("lib.kscd_sparse_decode.argtypes")]
    stub = re.findall(r'\("(\w+)",', body)
    assert stub == [f[0] for f in _lib.DecodeParams._fields_]


def test_append_kv_rejects_positions_outside_the_cache(lib):
    from paper_2512_16391_b200 import _lib
    from paper_2512_16391_b200.exceptions import InvalidArgumentError
    p = _lib.AppendKvParams(num_layers=1, batch=1, num_kv_heads=1, head_dim=128, position=16, kv_new=16,
                            k_caches=16, v_caches=16, kv_stride_batch=128, kv_stride_head=128,
                            cache_capacity=16)
    with pytest.raises(InvalidArgumentError, match="outside the cache"):
        _lib.call("kscd_append_kv", p, 0)
    p.cache_capacity = 0
    with pytest.raises(InvalidArgumentError, match="cache_capacity"):
        _lib.call("kscd_append_kv", p, 0)
