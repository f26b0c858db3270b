"""The C-ABI library loads on a CPU-only box and exports every symbol the
header declares (no compute calls)."""

import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _header_symbols():
    text = (ROOT / "include" / "lookahead_b200.h").read_text()
    return sorted(set(re.findall(r"\b(la_[a-z_0-9]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2402_02057_b200 import _build, _lib
    _build.build()
    return _lib.load()


def test_header_symbols_exported(lib):
    syms = _header_symbols()
    assert "la_decode_lookahead" in syms and len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s


def test_python_binding_covers_header(lib):
    from paper_2402_02057_b200 import _lib
    assert set(_header_symbols()) == set(_lib.EXPORTS)


def test_weight_names_and_abi(lib):
    import ctypes as C
    from paper_2402_02057_b200 import _lib
    assert lib.la_abi_version() == _lib.ABI_VERSION == 2
    d = _lib.la_model_desc(_lib.ARCH_LLAMA_BF16, 32000, 4096, 32, 32, 32, 128, 11008, 1e4, 1e-5, 2048)
    n = lib.la_weight_count(C.byref(d))
    assert n == 3 + 6 * 32
    names = [lib.la_weight_name(C.byref(d), i).decode() for i in range(n)]
    assert names[:3] == ["embed", "lm_head_tiles", "final_norm"]
    assert names[3:9] == ["0.wqkv_tiles", "0.wo_tiles", "0.wgu_tiles", "0.wd_tiles",
                          "0.attn_norm", "0.mlp_norm"]
    f = _lib.la_model_desc(_lib.ARCH_LLAMA_F32, 64, 64, 2, 4, 2, 16, 96, 1e4, 1e-5, 256)
    assert lib.la_weight_count(C.byref(f)) == 3 + 9 * 2
    assert lib.la_packed_bytes(32000, 4096) == 250 * 64 * 16384
    # 32016 rows -> 251 tiles, rounded up to the 2 tiles of one stream-K unit
    assert lib.la_packed_bytes(32016, 4096) == 252 * 64 * 16384
    g = _lib.la_model_desc(_lib.ARCH_GPT_F32, 256, 16, 2, 2, 2, 8, 64, 1e4, 1e-5, 256)
    assert lib.la_weight_count(C.byref(g)) == 4 + 12 * 2


def test_create_rejects_bad_descriptor_without_gpu(lib):
    import ctypes as C
    from paper_2402_02057_b200 import _lib
    d = _lib.la_model_desc(_lib.ARCH_LLAMA_BF16, 0, 4096, 32, 32, 32, 128, 11008, 1e4, 1e-5, 2048)
    out = C.c_void_p()
    rc = lib.la_create(C.byref(d), None, 0, 0, C.byref(out))
    assert rc == _lib.LA_ERR_INVALID_CONFIG
    assert b"positive" in lib.la_last_error() or b"weight" in lib.la_last_error()
