"""The drop-in boundary: libcovap_b200.so loads, exports every entry point
declared in include/covap_c.h, keeps the oracle out of the product, and
refuses to compute without a GPU (no CPU fallback)."""
import os
import re
import subprocess

import pytest

from conftest import ROOT, has_gpu

HEADER = os.path.join(ROOT, "include", "covap_c.h")
LIB = os.path.join(ROOT, "paper_2311_04499_b200", "libcovap_b200.so")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(covap_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("covap_plan_create", "covap_state_create", "covap_filter_pack", "covap_unpack",
                 "covap_sync_step", "covap_bucket_ready", "covap_allreduce", "covap_ccr",
                 "covap_choose_interval", "covap_profile_ccr", "covap_comm_create"):
        assert must in names


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (covap_[a-z0-9_]+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing


def test_ctypes_binding_covers_header():
    from paper_2311_04499_b200 import _lib
    assert sorted(_lib.EXPORTED) == declared()
    _lib.lib()  # binds every symbol with its signature


def test_product_does_not_link_the_oracle():
    out = subprocess.run(["nm", "-D", LIB], capture_output=True, text=True, check=True).stdout
    assert "oc_" not in " ".join(re.findall(r"\b(oc_\w+)", out))
    assert "ref_" not in " ".join(re.findall(r" T (ref_\w+)", out))
    ldd = subprocess.run(["ldd", LIB], capture_output=True, text=True).stdout
    assert "covap_oracle" not in ldd and "covap_ref" not in ldd
    src = os.path.join(ROOT, "paper_2311_04499_b200")
    for dirpath, _, files in os.walk(src):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".h", ".hpp")):
                body = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in body and "from oracle" not in body, f
                assert "covap_oracle" not in body, f


def test_kernels_are_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu(covap):
    plan = covap.plan_for(covap.load_layout("resnet50"), covap.CovapConfig(interval=4))
    with pytest.raises(covap.NoDeviceError):
        covap.CompressorState(plan)
    import ctypes
    from paper_2311_04499_b200 import _lib
    with pytest.raises(covap.Error):
        _lib.lib().covap_generate(ctypes.c_void_p(16), 4, 0, 1, 0, 0, None)
