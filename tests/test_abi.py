"""The C-ABI library loads on a CPU-only box and exports every symbol include/*.h declares."""
import os
import re

from paper_2503_17707_b200 import _binding as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    names = set()
    for h in ("pipeboost.h", "pipeboost_ops.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        names |= set(re.findall(r"PB_API\s+[\w\s\*]+?\b(pb_\w+)\s*\(", src))
    return names


def test_every_declared_symbol_is_exported_and_bound():
    lib = B.lib()
    names = declared()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), n
    assert names == set(B.declared_symbols()), names ^ set(B.declared_symbols())


def test_last_error_is_thread_local_string():
    try:
        B.pb_plan_create(None.__class__, (), 1, B.plan_opts())
    except Exception:
        pass
    assert isinstance(B.lib().pb_last_error(), bytes)


def test_library_is_sm100a():
    so = B.LIB_PATH
    data = open(so, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data
