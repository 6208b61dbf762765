"""CPU checks of the drop-in boundary: the C-ABI library loads and exports
every entry point include/gmcp_b200.h and include/gmcp_solver.h declare (no
compute without a GPU)."""
import ctypes as C
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gmcp_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2605_24339_b200 import gmcp
    lib = gmcp.library()
    names = _declared("gmcp_b200.h")
    assert len(names) >= 25
    solver = _declared("gmcp_solver.h")
    assert len(solver) >= 15
    missing = [n for n in names + solver if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a_cuda():
    """The shipped .so carries sm_100a SASS (cuobjdump), not a CPU build."""
    import shutil
    import subprocess
    from paper_2605_24339_b200 import gmcp
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([tool, "--list-elf", gmcp.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cuda_device_fails_loudly():
    """Without a GPU, context creation reports GMCP_ERR_CUDA (no CPU fallback)."""
    from paper_2605_24339_b200 import gmcp
    n = C.c_int(0)
    rc = gmcp.library().gmcp_device_count(C.byref(n))
    if rc == 0 and n.value > 0:
        return  # running on a GPU box: nothing to check here
    import pytest
    with pytest.raises(gmcp.GmcpCudaError):
        gmcp.Context(0)
