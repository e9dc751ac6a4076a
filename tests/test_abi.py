"""The C-ABI library builds, loads and exports every symbol include/bvss.h
declares; without an sm_100 device it fails loudly (no CPU fallback).
No compute calls (-m "not gpu")."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2412_03301_b200 import build
    return build.build()


def test_header_symbols_exported(libpath):
    hdr = open(os.path.join(ROOT, "include", "bvss.h")).read()
    declared = set(re.findall(r"BVSS_API\s+[\w\s\*]+?\b(bvss_\w+)\s*\(", hdr))
    assert len(declared) >= 20
    lib = ctypes.CDLL(libpath)
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    from paper_2412_03301_b200 import bvss
    assert set(bvss.EXPORTS) == declared


def test_no_cpu_fallback(libpath):
    import torch
    from paper_2412_03301_b200 import bvss
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the -m gpu tests")
    assert bvss.device_count() == 0
    import numpy as np
    with pytest.raises(bvss.BvssError) as e:
        bvss.Index(np.zeros((4, 8), np.float32), np.array([0, 4]), m=32, s=2, L=4)
    assert e.value.code in (bvss.EUNSUPPORTED, bvss.ECUDA)
