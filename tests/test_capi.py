"""The C-ABI library loads without a GPU and exports every symbol
include/chunkflow_b200.h declares; the product never touches oracle/."""
import os
import re
import subprocess

import paper_2503_02356_b200 as cf
from paper_2503_02356_b200 import capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "chunkflow_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cf_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    out = subprocess.run(["nm", "-D", "--defined-only", capi.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(cf_\w+)", out))
    declared = _declared()
    assert declared, "no declarations parsed"
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    assert sorted(capi.EXPORTS) == declared


def test_library_loads_and_reports_version():
    assert b"sm_100a" in cf.lib().cf_version()


def test_kernels_are_sm100a_tcgen05():
    """The shipped cubin is sm_100a and the GEMM issues tcgen05 MMAs fed by TMA."""
    out = subprocess.run(["cuobjdump", "-sass", capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "UTCHMMA" in out and "UTMALDG" in out and "LDTM" in out


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2503_02356_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".hpp", ".h", ".cuh")):
                text = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in text.replace("oracle/", "").lower() or f == "api.py", f


def test_context_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        return
    try:
        cf.Context(0)
    except capi.CfError as e:
        assert e.code in (1, 4)
    else:
        raise AssertionError("context creation must fail without a B200")
