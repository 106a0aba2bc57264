"""C-ABI library checks that need no GPU: it builds for sm_100a, loads, exports every
symbol include/hap.h declares, and its ctypes struct layouts match the header."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "hap.h")
HEADERS = sorted(os.path.join(ROOT, "include", f) for f in os.listdir(os.path.join(ROOT, "include"))
                 if f.endswith(".h"))


@pytest.fixture(scope="module")
def libhap():
    from paper_2605_08048_b200 import build
    build.build()
    import paper_2605_08048_b200 as hap
    return hap


def declared_functions():
    src = "\n".join(open(h).read() for h in HEADERS)
    return sorted(set(re.findall(r"^HAP_API\s+[\w\s\*]+?\b(hap_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("hap_create", "hap_destroy", "hap_sync", "hap_last_error", "hap_align",
                 "hap_permtest", "hap_permtest_batch", "hap_pvalue"):
        assert must in names


def test_library_exports_every_declared_symbol(libhap):
    out = subprocess.check_output(["nm", "-D", "--defined-only", libhap.LIB_PATH]).decode()
    exported = set(re.findall(r"\bT\s+(hap_\w+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    L = libhap.lib()
    for n in declared_functions():
        assert hasattr(L, n)


def test_sm100a_code_in_library(libhap):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                                   libhap.LIB_PATH]).decode()
    assert "sm_100a" in out


def test_tcgen05_and_tma_in_sass(libhap):
    """The GEMM kernel really uses tcgen05 (UTCHMMA), TMEM loads (LDTM) and TMA (UTMALDG)."""
    sass = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "-sass",
                                    libhap.LIB_PATH]).decode()
    for mn in ("UTCHMMA", "LDTM", "UTMALDG"):
        assert mn in sass, mn


def test_struct_layouts_match_header(libhap, tmp_path):
    """Compile a tiny C program against include/hap.h and compare sizeof/offsetof with
    the ctypes mirrors used by the binding."""
    prog = tmp_path / "lay.c"
    prog.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "hap.h"\n'
        'int main(){printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(hap_align_info),'
        ' offsetof(hap_align_info,t_obs), offsetof(hap_align_info,bad_row),'
        ' sizeof(hap_perm_cfg), offsetof(hap_perm_cfg,tie_rel), sizeof(hap_counts));}\n')
    exe = tmp_path / "lay"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(prog), "-o", str(exe)])
    got = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    want = [ctypes.sizeof(libhap.hap_align_info), libhap.hap_align_info.t_obs.offset,
            libhap.hap_align_info.bad_row.offset, ctypes.sizeof(libhap.hap_perm_cfg),
            libhap.hap_perm_cfg.tie_rel.offset, ctypes.sizeof(libhap.hap_counts)]
    assert got == want


def test_host_only_calls(libhap):
    """hap_pvalue is pure host arithmetic; hap_create refuses without an
    sm_100 device (no CPU fallback)."""
    assert libhap.hap_pvalue(0, 99) == 0.01
    assert libhap.hap_pvalue(49, 99) == 0.5
    assert libhap.hap_abi_version() == 1
    import torch
    if not torch.cuda.is_available():
        with pytest.raises(libhap.HapError):
            libhap.hap_create(0)


def test_product_never_imports_oracle():
    """The product package and its sources never reference the oracle."""
    pkg = os.path.join(ROOT, "paper_2605_08048_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "hap_oracle" not in txt, f
