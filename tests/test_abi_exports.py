"""The C-ABI library builds, loads, and exports every symbol include/eg.h
declares -- no compute calls (no GPU needed)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "eg.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(eg_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2303_02724_b200 import build
    return build.build()


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ["eg_create", "eg_compute", "eg_get_graph", "eg_get_labels", "eg_destroy", "eg_last_error"]:
        assert s in syms


def test_library_exports_every_declared_symbol(libpath):
    L = C.CDLL(libpath)
    for s in declared_symbols():
        assert hasattr(L, s), s
    out = subprocess.check_output(["nm", "-D", "--defined-only", libpath]).decode()
    exported = set(re.findall(r"\bT (eg_[a-z_0-9]+)\b", out))
    assert set(declared_symbols()) <= exported
    from paper_2303_02724_b200 import _abi
    assert set(_abi.EXPORTS) == set(declared_symbols())


def test_library_is_sm100a(libpath):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath]).decode()
    assert "sm_100a" in out


def test_struct_layouts_match_header(libpath):
    # compile a tiny C program against include/eg.h and compare sizeof/offsetof
    # with the ctypes mirrors in _abi.py
    from paper_2303_02724_b200 import _abi
    prog = r'''
#include <stdio.h>
#include <stddef.h>
#include "eg.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu\n", sizeof(eg_grid), sizeof(eg_csr), sizeof(eg_domain), sizeof(eg_graph), sizeof(eg_stats));
  printf("%zu %zu %zu\n", offsetof(eg_domain, csr), offsetof(eg_stats, jump_rounds), offsetof(eg_stats, bytes_alg));
  return 0; }
'''
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        cpath = os.path.join(td, "t.c")
        open(cpath, "w").write(prog)
        exe = os.path.join(td, "t")
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", exe, cpath])
        lines = subprocess.check_output([exe]).decode().split("\n")
    sizes = [int(x) for x in lines[0].split()]
    offs = [int(x) for x in lines[1].split()]
    assert sizes == [C.sizeof(_abi.EgGrid), C.sizeof(_abi.EgCsr), C.sizeof(_abi.EgDomain), C.sizeof(_abi.EgGraph),
                     C.sizeof(_abi.EgStats)]
    assert offs == [_abi.EgDomain.csr.offset, _abi.EgStats.jump_rounds.offset, _abi.EgStats.bytes_alg.offset]


def test_no_cpu_fallback_without_gpu(libpath):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2303_02724_b200 import _abi
    L = _abi.lib()
    h = C.c_void_p()
    assert L.eg_create(C.byref(h), 0, None) == _abi.EG_ERR_CUDA
    import paper_2303_02724_b200 as eg
    with pytest.raises(eg.EgError):
        eg.Context()


def test_product_package_does_not_touch_the_oracle():
    # the product path must never import / link / execute oracle/ (test infra)
    pkg = os.path.join(ROOT, "paper_2303_02724_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".h", ".cpp")):
                src = open(os.path.join(dirpath, fn)).read()
                assert "import oracle" not in src and "from oracle" not in src, fn
                assert "eg_oracle" not in src and "ego_" not in src, fn
