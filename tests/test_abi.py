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
    with pytest.raises(bvss.BvssError) as e:  # the multi-device group too (every shard build fails loudly)
        bvss.Group(np.zeros((4, 8), np.float32), np.array([0, 2, 4]), devices=[0, 0], m=32, s=2, L=4)
    assert e.value.code in (bvss.EUNSUPPORTED, bvss.ECUDA)
    with pytest.raises(bvss.BvssError) as e:
        bvss.Group(np.zeros((4, 8), np.float32), np.array([0, 2, 4]), devices=[], m=32, s=2, L=4)
    assert e.value.code == bvss.EINVAL


@pytest.mark.parametrize("struct,pyname", [("bvss_params", "Params"), ("bvss_info", "Info"), ("bvss_stats", "Stats")])
def test_struct_layouts_match_header(tmp_path, struct, pyname):
    """The ctypes mirrors of the ABI structs have the header's size and field offsets (compiled with gcc)."""
    import shutil
    import subprocess
    from paper_2412_03301_b200 import bvss
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    py = getattr(bvss, pyname)
    fields = [f for f, _ in py._fields_]
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "bvss.h"\nint main(void) {\n'
                   f'  printf("%zu\\n", sizeof({struct}));\n' +
                   "".join(f'  printf("%zu\\n", offsetof({struct}, {f}));\n' for f in fields) + "  return 0;\n}\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = [int(x) for x in subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()]
    assert out[0] == ctypes.sizeof(py), (struct, out[0], ctypes.sizeof(py))
    assert out[1:] == [getattr(py, f).offset for f in fields]
