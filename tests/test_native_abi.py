"""The C-ABI library exists, loads without a GPU and exports every declared symbol."""

import ctypes
import os
import subprocess

from paper_2410_00425_b200 import _native


def test_library_built():
    assert os.path.exists(_native.LIB_PATH), "run python -m paper_2410_00425_b200.build_native"


def test_exports_every_header_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    _native.load()  # binds the struct-taking entry points too (cabi)
    declared = _native.header_symbols()
    assert len(declared) >= 12
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    # and the ctypes table binds exactly the declared set
    assert set(_native._SIGNATURES) == set(declared)


def test_abi_version_and_sm100a_cubin():
    lib = _native.load()
    assert lib.bs_abi_version() == _native.ABI_VERSION
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_product_never_imports_the_oracle():
    """The oracle is test infrastructure: the product package has no path into it (and hence
    no CPU fallback through it)."""
    import ast
    import os

    pkg = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2410_00425_b200")
    for fn in os.listdir(pkg):
        if not fn.endswith(".py"):
            continue
        tree = ast.parse(open(os.path.join(pkg, fn)).read())
        for node in ast.walk(tree):
            if isinstance(node, ast.Import):
                assert not any(a.name.split(".")[0] == "oracle" for a in node.names), fn
            if isinstance(node, ast.ImportFrom) and node.level == 0:
                assert (node.module or "").split(".")[0] != "oracle", fn
