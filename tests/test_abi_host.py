"""The C-ABI library loads and exports every symbol include/sldg.h declares; host-only
helpers work without a GPU; the product package never touches the oracle."""
import ast
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "sldg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sldg_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    from paper_1603_07008_b200 import sldg
    return sldg.lib()


def test_every_declared_symbol_is_exported(lib):
    names = header_functions()
    assert len(names) >= 20
    out = subprocess.check_output(["nm", "-D", "--defined-only",
                                   os.path.join(ROOT, "paper_1603_07008_b200", "libsldg.so")]).decode()
    exported = set(re.findall(r" T (sldg_[a-z0-9_]+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    from paper_1603_07008_b200 import sldg
    assert sorted(sldg.EXPORTS) == names


def test_library_is_sm100a(lib):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                                   os.path.join(ROOT, "paper_1603_07008_b200", "libsldg.so")]).decode()
    assert "sm_100a" in out


def test_halo_widths_and_owner(lib):
    from paper_1603_07008_b200 import sldg
    # lines read layers i - i* - 1 and i - i* (P:259-268): i* in [imin, imax]
    assert sldg.halo_widths(0, 0) == (1, 0)
    assert sldg.halo_widths(-1, 0) == (1, 1)
    assert sldg.halo_widths(-3, -2) == (0, 3)
    assert sldg.halo_widths(2, 5) == (6, 0)
    # balanced block split: 10 layers over 4 ranks -> 3,3,2,2
    owners = [sldg.layer_owner(10, 4, l) for l in range(10)]
    assert owners == [(0, 0), (0, 1), (0, 2), (1, 0), (1, 1), (1, 2), (2, 0), (2, 1), (3, 0), (3, 1)]
    with pytest.raises(sldg.SldgError):
        sldg.layer_owner(10, 4, 10)


def test_create_without_gpu_fails_cleanly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_1603_07008_b200 import Grid, SldgError
    with pytest.raises(SldgError):
        Grid([8, 8], 2)
    with pytest.raises(SldgError):  # validation happens before any device call
        Grid([8, 0], 2)


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1603_07008_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                tree = ast.parse(open(os.path.join(dirpath, f)).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert all(not a.name.startswith("oracle") for a in node.names), f
                    if isinstance(node, ast.ImportFrom):
                        assert not (node.module or "").startswith("oracle"), f
            if f.endswith((".cu", ".h", ".cuh", ".cpp")):
                incs = re.findall(r"#include\s*[<\"]([^>\"]+)", open(os.path.join(dirpath, f)).read())
                assert not any("oracle" in i for i in incs), f
    # and the oracle never includes the product's headers
    incs = re.findall(r"#include\s*[<\"]([^>\"]+)", open(os.path.join(ROOT, "oracle", "sldg_oracle.c")).read())
    assert sorted(incs) == ["math.h", "stdint.h", "stdlib.h", "string.h"]
