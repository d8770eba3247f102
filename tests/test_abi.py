"""The C-ABI library loads and exports every symbol include/gsm.h declares
(no compute calls without a GPU); without a device the library fails loudly
(GSM_ERR_NO_DEVICE) instead of falling back to the CPU."""
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2003_01527_b200 import gsm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "gsm.h")).read()
    return sorted(set(re.findall(r"GSM_API\s+[\w\s\*]*?\b(gsm_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared()
    for n in ["gsm_load_graph", "gsm_match", "gsm_free", "gsm_result_free", "gsm_last_error"]:
        assert n in names
    assert set(names) == set(gsm.EXPORTS)


def test_library_exports_every_declared_symbol():
    out = subprocess.check_output(["nm", "-D", "--defined-only", gsm.SO_PATH], text=True)
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    L = gsm.lib()
    for n in declared():
        assert hasattr(L, n)
    assert b"sm_100a" in L.gsm_version()


def test_sm100a_code_in_library():
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", gsm.SO_PATH], text=True)
    assert "sm_100a" in out


def test_no_cpu_fallback_without_device():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is visible")
    except ImportError:
        pass
    off = np.array([0, 1, 2], np.int64)
    cols = np.array([1, 0], np.int32)
    with pytest.raises(gsm.GsmError) as e:
        gsm.gsm_load_graph(2, off, cols)
    assert e.value.status == 6  # GSM_ERR_NO_DEVICE


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2003_01527_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "oracle.h" not in txt, f
