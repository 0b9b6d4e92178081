"""C-ABI checks that need no GPU: the library builds for sm_100a, loads, exports every
function include/autx.h declares, and the ctypes structs have the C layout (checked by
compiling a tiny C program against the header with gcc)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "autx.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2502_13965_b200 import _build
    _build.build()
    from paper_2502_13965_b200.autx import load_library
    return load_library()


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(autx_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    names = declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), f"{n} declared in autx.h but not exported"
    from paper_2502_13965_b200.autx import exported_symbols
    assert sorted(exported_symbols()) == names


def test_sm100a_code_only(lib):
    from paper_2502_13965_b200._build import LIB
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_struct_layout_matches_header(tmp_path, lib):
    from paper_2502_13965_b200 import autx as A
    c = tmp_path / "sz.c"
    c.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "autx.h"\nint main(){printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu\\n",'
                 'sizeof(autx_config), sizeof(autx_call_desc), sizeof(autx_step_out), sizeof(autx_kv_layout),'
                 'sizeof(autx_swap_stats), sizeof(autx_call_state), sizeof(autx_step_timing), offsetof(autx_config, stream), sizeof(autx_selection_stats));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.dirname(HEADER), str(c), "-o", str(exe)])
    got = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    want = [ctypes.sizeof(A.Config), A.CALL_DESC.itemsize, ctypes.sizeof(A.StepOut),
            ctypes.sizeof(A.KvLayout), ctypes.sizeof(A.SwapStats), A.CALL_STATE.itemsize,
            ctypes.sizeof(A.StepTiming), A.Config.stream.offset, ctypes.sizeof(A.StepStats)]
    assert got == want


def test_version_and_no_gpu_create_fails_loudly(lib):
    assert b"sm_100a" in lib.autx_version()
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2502_13965_b200 import Scheduler, AutxError
    with pytest.raises(AutxError):
        Scheduler(policy="plas", K=1, quanta=(None,), max_batch=2)


def test_product_does_not_import_oracle():
    """The product path never imports the oracle (task rule: no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2502_13965_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b|importlib.*oracle", src, re.M), f
            if f.endswith((".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"#include\s+[<\"].*oracle", src), f
