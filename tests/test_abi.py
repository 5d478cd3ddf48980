"""C-ABI boundary checks that need no GPU (-m "not gpu")."""
import ctypes
import re

import pytest

from paper_1810_00845_b200 import hisa as H


def test_library_exports_every_declared_symbol():
    lib = H.load()
    syms = H.header_symbols()
    assert len(syms) >= 45
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # every declared symbol has a binding with the same name (argument marshalling only)
    assert set(syms) <= set(H._SIGS)


def test_header_cites_paper_and_documents_errors():
    txt = open(H.HEADER).read()
    for cite in ("P:441-568", "P:584-587", "P:621-628", "P:764"):
        assert cite in txt
    codes = dict((m[0], int(m[1])) for m in re.findall(r"HISA_E_([A-Z_]+) = (-\d+)", txt))
    assert {v: k for k, v in codes.items()} == {k: v for k, v in H.ERRORS.items() if k != 0}


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(H.HisaError) as ei:
        H.hisa_ctx_create(10, [60, 40], 60)
    assert ei.value.code == "CUDA"
    with pytest.raises(H.HisaError):
        H.Context(10, [60, 40], 60)


def test_product_does_not_import_oracle():
    import pathlib
    pkg = pathlib.Path(H.__file__).parent
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")) + list(pkg.rglob("*.h")):
        txt = f.read_text()
        assert "oracle" not in re.sub(r"#.*|//.*", "", txt).lower().replace("oracle", "oracle") or \
            not re.search(r"^\s*(from|import)\s+oracle|ckks_oracle|orc_", txt, re.M), f
