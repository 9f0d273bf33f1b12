"""The C-ABI library loads without a GPU and exports exactly what
include/msinfer.h declares; the product path has no CPU fallback."""

import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "msinfer.h")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(msi_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2504_02263_b200 import _lib
    return _lib.load(build_if_missing=True)


def test_header_symbols_exported(lib):
    names = declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), f"{n} declared in msinfer.h but not exported"
    out = subprocess.run(["nm", "-D", "--defined-only", lib._name], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (msi_\w+)", out))
    assert exported == set(names), f"extra/missing exports: {exported ^ set(names)}"


def test_python_binding_covers_header(lib):
    from paper_2504_02263_b200 import _lib
    assert set(_lib.exported_symbols()) == set(declared())


def test_library_is_sm100a_only(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", lib._name], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(8\d|9\d|120)\b", out)


def test_tcgen05_and_tma_in_sass(lib):
    sass = subprocess.run(["cuobjdump", "-sass", lib._name], capture_output=True, text=True).stdout
    for mnem in ("UTCHMMA", "UTMALDG", "LDTM"):
        assert mnem in sass, f"{mnem} missing: expert GEMM is not on tcgen05/TMA"


def test_no_gpu_calls_fail_loudly(lib):
    """Without a GPU the product path raises instead of falling back."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2504_02263_b200 import _lib
    with pytest.raises(_lib.MsiError):
        _lib.call("msi_check_device")


def test_oracle_not_linked_into_product(lib):
    out = subprocess.run(["nm", "-D", lib._name], capture_output=True, text=True).stdout
    assert "orc_" not in out
    for f in os.listdir(os.path.join(ROOT, "paper_2504_02263_b200")):
        if f.endswith(".py"):
            src = open(os.path.join(ROOT, "paper_2504_02263_b200", f)).read()
            assert "import oracle" not in src and "from oracle" not in src, f
