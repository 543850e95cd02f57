"""CPU-side checks of the C-ABI library (no compute calls: no GPU here).

* libdyq.so builds for sm_100a and loads;
* it exports every function include/dyq.h declares;
* synchronous argument validation (pure host logic) returns the documented
  status codes before anything touches a device;
* the product package never imports the oracle (and vice versa).
"""
import ast
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "dyq.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"DYQ_API\s+[\w\s\*]+?\b(dyq_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    from paper_2603_07904_b200 import build
    build.build()
    from paper_2603_07904_b200 import dyq
    return dyq


def test_header_declares_the_boundary():
    fns = _header_functions()
    for f in ("dyq_pack_weights", "dyq_select_bits", "dyq_qlinear", "dyq_qlinear_i32_partials"):
        assert f in fns


def test_library_exports_every_header_symbol(L):
    lib = L.lib()
    missing = [f for f in _header_functions() if not hasattr(lib, f)]
    assert not missing, missing
    # and the Python binding covers every one of them
    assert set(_header_functions()) <= set(L._SIGS)


def test_library_is_sm100a(L):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", L.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_sync_validation(L):
    WD = L.WDesc
    with pytest.raises(L.DyqError) as e:
        L.pack_weights_size(WD(16, 64, 64, 3, 0))
    assert e.value.code == 1  # EINVAL wbits
    with pytest.raises(L.DyqError) as e:
        L.pack_weights_size(WD(24, 64, 64, 4, 0))
    assert e.value.code == 2  # N % 16
    with pytest.raises(L.DyqError) as e:
        L.pack_weights_size(WD(16, 96, 64, 4, 0))
    assert e.value.code == 2  # K % G
    with pytest.raises(L.DyqError) as e:
        L.pack_weights_size(WD(16, 64, 32, 4, 0))
    assert e.value.code == 2  # G in {64,128}
    cb, mb = L.pack_weights_size(WD(4096, 4096, 64, 4, 0))
    assert cb == 4096 * 4096 // 2 and mb >= 4096 * 64 * 5
    cb8, _ = L.pack_weights_size(WD(4096, 4096, 64, 8, 0))
    assert cb8 == 4096 * 4096
    bad = L.default_calib(theta_24=0.4, theta_48=0.3)
    with pytest.raises(L.DyqError) as e:
        L.state_size(4, bad)
    assert e.value.code == 1
    assert L.state_size(64, L.default_calib()) < 64 * (64 * 1024)  # < 64 KB per stream


def test_product_and_oracle_are_independent():
    """Neither side imports the other."""
    def imports(path):
        tree = ast.parse(open(path).read())
        names = set()
        for node in ast.walk(tree):
            if isinstance(node, ast.Import):
                names |= {a.name.split(".")[0] for a in node.names}
            elif isinstance(node, ast.ImportFrom) and node.module:
                names.add(node.module.split(".")[0])
        return names
    pkg = os.path.join(ROOT, "paper_2603_07904_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            assert "oracle" not in imports(os.path.join(pkg, f)), f
    for f in os.listdir(os.path.join(pkg, "csrc")):
        text = open(os.path.join(pkg, "csrc", f)).read()
        assert not re.search(r'#include\s*[<"][^>"]*(oracle|dyq_ref)', text), f
    assert "paper_2603_07904_b200" not in imports(os.path.join(ROOT, "oracle", "__init__.py"))
    assert "dyq.h" not in open(os.path.join(ROOT, "oracle", "dyq_ref.c")).read()
