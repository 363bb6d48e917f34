"""The C-ABI library loads (no GPU needed) and exports every symbol include/*.h declares."""
import re
from pathlib import Path

from paper_2201_11990_b200 import _native

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[\w\s\*]+?\b(mt_\w+)\s*\(", text, flags=re.M):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    names = declared_symbols()
    assert len(names) > 40
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding declares exactly the header's functions
    assert set(_native.EXPORTED) == names


def test_version_and_error_string():
    lib = _native.lib()
    assert b"sm_100a" in lib.mt_version()
    import ctypes as C
    rc = lib.mt_pipeline_efficiency(0, 4, C.byref(C.c_double()))
    assert rc == 1 and b"micro_batches" in lib.mt_last_error()


def test_example_caller_compiles_against_the_header():
    """examples/train_lm.cpp (the C++ binding INTEGRATION.md describes: planner types, stage, vocab,
    blend feed, optimizer) must compile against include/mtnlg.h as documented."""
    import shutil
    import subprocess
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    if shutil.which("g++") is None:
        import pytest
        pytest.skip("no g++")
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra", f"-I{root / 'include'}",
                        "-I/usr/local/cuda/include", str(root / "examples" / "train_lm.cpp")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
