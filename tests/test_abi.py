"""The C-ABI library loads without a GPU and exports exactly what
include/flexshm.h declares; the package never imports the oracle; the
product path refuses to run without the native library."""

from __future__ import annotations

import ast
import os
import re
import subprocess

from paper_2511_09143_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "flexshm.h")
PKG = os.path.join(ROOT, "paper_2511_09143_b200")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(fmx_\w+)\s*\(", text, re.M)))


def test_every_declared_symbol_is_exported():
    names = declared()
    assert len(names) >= 18
    L = _lib.lib()
    for name in names:
        assert hasattr(L, name), name
    assert sorted(_lib.EXPORTS) == names
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    for name in names:
        assert re.search(rf"\bT {name}\b", out), f"{name} not a defined text symbol"


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out, out


def test_abi_version():
    assert _lib.lib().fmx_abi_version() == 1


def test_product_package_never_imports_the_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if not f.endswith(".py"):
                continue
            tree = ast.parse(open(os.path.join(dirpath, f)).read())
            for node in ast.walk(tree):
                if isinstance(node, ast.Import):
                    assert not any(a.name.split(".")[0] == "oracle" for a in node.names), f
                if isinstance(node, ast.ImportFrom):
                    assert (node.module or "").split(".")[0] != "oracle", f


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    import pytest
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "libflexshm.so"))
    with pytest.raises(ImportError):
        _lib.lib()


def test_collectives_refuse_cpu_tensors():
    import pytest
    import torch
    from paper_2511_09143_b200.comm import ShmCommunicator, _check_tensor
    with pytest.raises(ValueError):
        _check_tensor(torch.zeros(4), "tensor")
    assert ShmCommunicator  # the class exists; a CPU tensor never reaches the C ABI
