"""CPU-only checks of the C-ABI library: it loads without a GPU, exports every
symbol include/gemm_f16.h declares, and rejects bad arguments before touching
a device (argument errors never need CUDA; no compute call is made here)."""
import ctypes
import os
import re

import pytest

import paper_2108_13191_b200 as g

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions(header="gemm_f16.h"):
    with open(os.path.join(ROOT, "include", header)) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:gemm_status_t|int|uint32_t|const char\*)\s+(\w+)\s*\(", text, re.M)))


def test_header_declares_expected_api():
    names = _declared_functions()
    assert set(names) == set(g.EXPORTED_SYMBOLS), names
    assert set(_declared_functions("gemm_f16_diag.h")) == set(g.DIAG_SYMBOLS)


def test_library_loads_and_exports_every_symbol():
    lib = g.load_library()
    declared = _declared_functions() + _declared_functions("gemm_f16_diag.h")
    for name in declared:
        assert hasattr(lib, name), name
    out = os.popen(f"nm -D --defined-only {g.library_path()}").read()
    for name in declared:
        assert re.search(rf"\bT {name}$", out, re.M), name


def test_public_options_carry_no_diagnostic_knobs():
    """the product struct holds no wrong-results or rejected knobs."""
    with open(os.path.join(ROOT, "include", "gemm_f16.h")) as f:
        text = f.read()
    body = text[text.index("typedef struct {"):text.index("} gemm_options_t;")]
    fields = re.findall(r"^\s*(?:int|const void\*|void\*)\s+(\w+);", body, re.M)
    assert fields == [f for f, _ in g._Options._fields_], fields
    for bad in ("debug_flags", "epi_pace", "k_serpentine", "wait_hint_ns", "c_row_prefetch", "trace"):
        assert bad not in fields


def test_stream_k_windows_never_overlap_at_the_wrap():
    """windows are whole and round robin, so any two launches fewer than
    pool/window apart -- in particular the two straddling the wrap -- get disjoint windows."""
    lib = g.load_library()
    win = lib.gemm_f16_diag_sk_window_slots()
    pool = lib.gemm_f16_diag_sk_pool_slots()
    assert pool % win == 0 and win >= 16 * 74   # 16 slots per cluster, 74 clusters on a B200
    n = pool // win
    for start in (0, n - 3, 2 ** 32 - 5, 12345):
        bases = [lib.gemm_f16_diag_sk_window_base((start + i) % 2 ** 32) for i in range(n)]
        assert all(b % win == 0 and b + win <= pool for b in bases)
        assert len(set(bases)) == n, (start, bases)


def test_status_strings():
    lib = g.load_library()
    for s, name in ((0, b"GEMM_OK"), (1, b"GEMM_ERR_INVALID_VALUE"), (2, b"GEMM_ERR_MISALIGNED"),
                    (3, b"GEMM_ERR_UNSUPPORTED_DEVICE"), (4, b"GEMM_ERR_CUDA")):
        assert lib.gemm_status_string(s) == name


def _call(M, N, K, A=16, lda=None, B=16, ldb=None, C=16, ldc=None, acc=0):
    lib = g.load_library()
    lda = K if lda is None else lda
    ldb = N if ldb is None else ldb
    ldc = N if ldc is None else ldc
    return lib.gemm_f16(M, N, K, A, lda, B, ldb, C, ldc, acc, None)


def test_argument_errors_without_gpu():
    # negative extents, short leading dims, bad mode, NULL with work: INVALID_VALUE
    assert _call(-1, 8, 8) == 1
    assert _call(8, -1, 8) == 1
    assert _call(8, 8, -1) == 1
    assert _call(8, 8, 8, lda=4) == 1
    assert _call(8, 8, 8, ldb=4) == 1
    assert _call(8, 8, 8, ldc=4) == 1
    assert _call(8, 8, 8, acc=2) == 1
    assert _call(8, 8, 8, A=0) == 1
    assert _call(1 << 31, 8, 8) == 1
    # misaligned pointers / leading dims: MISALIGNED
    assert _call(8, 8, 8, A=18) == 2
    assert _call(8, 8, 12) == 2                 # lda*2 = 24 bytes
    assert _call(8, 12, 8, ldb=12, ldc=12) == 2 # ldb*2 = 24 bytes
    assert _call(8, 6, 8, ldb=8, ldc=6) == 2    # F32 ldc*4 = 24 bytes
    # quick returns: nothing launched, no device needed
    assert _call(0, 8, 8) == 0 and g.last_launches() == 0
    assert _call(8, 0, 8, ldb=8, ldc=8) == 0
    assert _call(8, 8, 0, lda=8) == 0


def test_config_info_is_host_only():
    for name, cid in g.CONFIGS.items():
        if cid == 0:
            continue
        for acc in (0, 1):
            info = g.config_info(cid, acc)
            assert info["tile_m"] == 128 * info["cta_group"]
            assert info["smem_bytes"] <= 232448
            assert info["stages"] >= 3
    with pytest.raises(g.GemmError):
        g.config_info(0)
    with pytest.raises(g.GemmError):
        g.config_info(99)


def test_config_names_match_the_header_enum():
    # the binding's config names are the header's gemm_config_t, value for value
    import os
    import re
    hdr = open(os.path.join(os.path.dirname(__file__), "..", "include", "gemm_f16.h")).read()
    enum = {m.group(1).lower(): int(m.group(2)) for m in re.finditer(r"GEMM_CFG_(\w+)\s*=\s*(\d+)", hdr)}
    count = enum.pop("count")
    assert enum.pop("auto") == 0 and g.CONFIGS.get("auto", 0) == 0
    named = {k: v for k, v in g.CONFIGS.items() if k != "auto"}
    assert named == enum
    assert sorted(enum.values()) == list(range(1, count))


def test_product_path_does_not_import_oracle():
    # the product package must never reach the oracle (no CPU fallback)
    pkg = os.path.join(ROOT, "paper_2108_13191_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".c")):
                with open(os.path.join(dirpath, fn)) as f:
                    src = f.read()
                assert not re.search(r"\bimport\s+oracle\b|from\s+oracle\b|liboracle", src), fn
