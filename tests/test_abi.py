"""The C-ABI boundary without a GPU: libgpuos_cuda.so loads, exports every
entry point include/gpuos_cuda.h declares, and the ctypes mirror of its
structs matches the header's layout."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gpuos_cuda.h")


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(gpuos_\w+)\s*\(", src, re.M)))


def test_header_declares_the_boundary():
    fns = declared_functions()
    assert len(fns) >= 50
    for must in ("gpuos_dev_open", "gpuos_ring_reserve", "gpuos_ring_publish", "gpuos_table_install_program",
                 "gpuos_table_kill", "gpuos_launch_task", "gpuos_jit_compile"):
        assert must in fns


def test_library_exports_every_declared_symbol():
    from paper_2604_17861_b200 import abi
    lib = abi.load_library()
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing
    assert set(abi.EXPORTS) == set(declared_functions())
    assert lib.gpuos_abi_version() == 1


def test_struct_layouts_and_error_names():
    from paper_2604_17861_b200 import abi
    lib = abi.load_library()
    assert C.sizeof(abi.View) == 48 and C.sizeof(abi.Task) == 384 and C.sizeof(abi.Instr) == 16
    assert abi.Task.scalars.offset == 64 and abi.Task.views.offset == 128
    for i, name in enumerate(abi.ERRORS):
        assert lib.gpuos_error_name(i).decode() == name
    cfg = abi.Cfg()
    assert lib.gpuos_default_cfg(C.byref(cfg)) == 0
    assert cfg.capacity == 4096 and cfg.table_slots == 1024 and cfg.spin_iterations == 64


def test_open_without_gpu_fails_loudly():
    """No CPU fallback: with no device the open call reports an error."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2604_17861_b200 import abi
    with pytest.raises(abi.GpuosError):
        abi.Device(0)
