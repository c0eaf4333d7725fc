"""CPU-side checks of the C ABI: the library builds, loads, and exports every
entry point declared in include/wavecell_b200.h (no compute calls here)."""

import re
from pathlib import Path

from paper_2501_19013_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "wavecell_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(wcb_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(_lib.EXPORTS)


def test_library_exports_every_symbol():
    lib = _lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.wcb_abi_version() == 2


def test_no_device_here_is_reported_not_faked():
    # On the CPU box there is no GPU: creating a context must fail loudly.
    if _lib.device_count() == 0:
        import pytest
        with pytest.raises(Exception):
            _lib.Context(0)
