"""The ctypes stub printed in INTEGRATION.md binds the same argument lists as
the library's own binding (paper_2504_02263_b200/_lib.py SIGNATURES)."""

import ctypes
import os
import re

from paper_2504_02263_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_integration_stub_matches_signatures():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = text.split("## 2. ctypes binding")[1].split("```python")[1].split("```")[0]
    ns = {"ctypes": ctypes}
    # evaluate only the argtypes lines against ctypes aliases (no library load)
    exec("P, I, U32 = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint32", ns)
    checked = 0
    for m in re.finditer(r"lib\.(msi_\w+)\.argtypes = (\[.*?\])", block, re.S):
        name, expr = m.group(1), m.group(2)
        if "msi_plan" in expr:  # the struct is declared in the stub itself
            continue
        got = eval(expr, ns)
        want = _lib.SIGNATURES[name][1]
        assert [t.__name__ if hasattr(t, "__name__") else t for t in got] == \
               [t.__name__ if hasattr(t, "__name__") else t for t in want], name
        checked += 1
    assert checked >= 7


def test_integration_stub_plan_struct_matches_library():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = text.split("## 2. ctypes binding")[1].split("```python")[1].split("```")[0]
    start = block.index("class msi_plan(ctypes.Structure):")
    lines = []
    for ln in block[start:].splitlines()[1:]:
        code = ln.split("#")[0].rstrip()
        lines.append(code.replace("_fields_ = ", "").strip())
        if code.endswith(")]"):
            break
    fields = eval(" ".join(lines), {"ctypes": ctypes})
    assert [f[0] for f in fields] == [f[0] for f in _lib.Plan._fields_]
    assert ctypes.sizeof(type("S", (ctypes.Structure,), {"_fields_": fields})) == ctypes.sizeof(_lib.Plan)
