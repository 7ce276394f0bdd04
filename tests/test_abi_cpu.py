"""CPU checks of the C-ABI boundary: libdvm.so loads, exports every symbol that
include/dvm.h declares, and rejects bad parameters with the documented status
codes before touching a GPU.  No compute calls (there is no GPU here)."""
import os
import re

import pytest
import torch

from paper_1201_3986_b200 import dvm

needs_no_gpu = pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure path")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "dvm.h")).read()
    return sorted(set(re.findall(r"DVM_API[^;(]*?\b(dvm_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = dvm.load()
    names = _declared()
    assert len(names) >= 16
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_abi_version_and_status_strings():
    lib = dvm.load()
    assert lib.dvm_abi_version() == 1
    for code, name in dvm.STATUS.items():
        assert lib.dvm_status_str(code).decode().startswith(name)


@pytest.mark.parametrize("args,status", [
    ((4, 16, 2, 0), "DVM_E_DIM"),
    ((1, 16, 2, 0), "DVM_E_DIM"),
    ((2, 16, 2, 1), "DVM_E_KERNEL"),
    ((3, 32, 2, 0), "DVM_E_KERNEL"),
    ((2, 24, 2, 0), "DVM_E_UNSUPPORTED"),
    ((3, 512, 2, 1), "DVM_E_UNSUPPORTED"),
    ((2, 16, 0, 0), "DVM_E_ORDER"),
])
def test_plan_validation(args, status):
    d, N, Nbar, kernel = args
    with pytest.raises(dvm.DvmError) as ei:
        dvm.Plan(d, N, Nbar, kernel=kernel)
    assert ei.value.name == status


def test_explicit_ntilde_and_shard_validation():
    with pytest.raises(dvm.DvmError) as ei:
        dvm.Plan(2, 16, 3, Ntilde=8)  # 2*8+1 > 16
    assert ei.value.name == "DVM_E_ORDER"
    with pytest.raises(dvm.DvmError) as ei:
        dvm.Plan(2, 16, 3, Ntilde=2)  # N̄ > Ñ
    assert ei.value.name == "DVM_E_ORDER"
    with pytest.raises(dvm.DvmError) as ei:
        dvm.Plan(2, 16, 3, shard_rank=2, shard_world=2)
    assert ei.value.name == "DVM_E_SHAPE"
    with pytest.raises(dvm.DvmError) as ei:
        dvm.Plan(2, 16, 3, L=-1.0)
    assert ei.value.name == "DVM_E_UNSUPPORTED"


@needs_no_gpu
def test_no_gpu_fails_loudly():
    # A valid plan on a machine without a GPU must raise, never fall back to CPU.
    with pytest.raises(dvm.DvmError) as ei:
        dvm.Plan(3, 32, 4)
    assert ei.value.name == "DVM_E_CUDA"
    with pytest.raises(dvm.DvmError) as ei:
        dvm.Plan(2, 16, 5)  # valid: Ñ = max(3, 5) = 5 and 2Ñ+1 <= 16, so it reaches CUDA
    assert ei.value.name == "DVM_E_CUDA"
