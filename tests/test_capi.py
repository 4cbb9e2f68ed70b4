"""The C-ABI drop-in boundary (include/moe_b200.h): the library loads, exports
every declared symbol, and -- with no CUDA device -- fails loudly instead of
falling back to the CPU."""
import ctypes
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol(moe):
    lib = moe.lib()
    declared = moe.exported_symbols()
    assert len(declared) >= 45
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    nm = subprocess.run(["nm", "-D", "--defined-only", moe.LIB_PATH], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in nm.splitlines() if " T " in ln}
    assert set(declared) <= exported


def test_library_is_sm100a_only(moe):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", moe.LIB_PATH], capture_output=True,
                         text=True).stdout
    arches = {ln.split(".")[-2] for ln in out.splitlines() if ".cubin" in ln}
    assert arches == {"sm_100a"}, arches


def test_product_does_not_link_the_oracle(moe):
    deps = subprocess.run(["ldd", moe.LIB_PATH], capture_output=True, text=True).stdout
    assert "moe_oracle" not in deps and "moeserve_ref" not in deps
    # no product source includes the oracle header or imports the oracle package
    for path, _, files in os.walk(os.path.join(ROOT, "paper_2407_14417_b200")):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".cuh", ".h", ".hpp")):
                text = open(os.path.join(path, f), errors="ignore").read()
                assert "moe_oracle.h" not in text and "libmoe_oracle" not in text, f
                assert "import oracle" not in text and "from oracle" not in text, f


def _has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_cuda(), reason="checks the no-device error path")
def test_kernels_fail_loudly_without_a_device(moe):
    with pytest.raises(moe.MoeError) as ei:
        moe.gate_topk(None, None, 1, 512, 8, 2, None, None, stream=0)
    assert ei.value.code == 1 and "no CUDA device" in str(ei.value)
    with pytest.raises(moe.MoeError):
        moe.MoeEngine(2, 8, 2, 512, 1792, moe.PlacementPlan([0] * 16, [0] * 16, 0))


def test_status_codes_mirror_cli(moe):
    # usage (2): bad shape before any device work
    with pytest.raises(moe.UsageError):
        moe.ffn(None, None, None, 1, 2, [], 512, 1792, None, 0, None, stream=0)
    # validation (3) / infeasible (4) from the planner
    with pytest.raises(moe.ValidationError):
        moe.make_plan(moe.TaskRequest(moe.QUALITY, None, 0), moe.HardwareProfile(10**11), moe.mixtral_sec41())
    with pytest.raises(moe.InfeasibleError):
        moe.make_plan(moe.TaskRequest(moe.THROUGHPUT, None, 0), moe.HardwareProfile(10**9), moe.mixtral_sec41())
