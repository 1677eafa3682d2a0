"""CPU-side checks of the boundary: libtfn.so builds for sm_100a, loads, exports every
symbol include/tfn.h declares, contains sm_100a SASS, and fails loudly (no CPU
fallback) without a GPU.  No compute calls here."""
import ctypes
import os
import re
import subprocess

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tfn.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tfn_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def so():
    from paper_2005_08165_b200 import build
    return build.build()


def test_header_declares_the_north_star_calls():
    d = _declared()
    for name in ("tfn_create", "tfn_estimate", "tfn_estimate_disparity", "tfn_destroy"):
        assert name in d


def test_library_exports_every_declared_symbol(so):
    L = ctypes.CDLL(so)
    for name in _declared():
        assert hasattr(L, name), name
    nm = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (tfn_[a-z_0-9]+)", nm))
    assert set(_declared()) <= exported
    from paper_2005_08165_b200.tfn import ABI_SYMBOLS
    assert set(ABI_SYMBOLS) == set(_declared())


def test_library_is_sm100a_native(so):
    out = subprocess.run(["cuobjdump", "-lelf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    full = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    parts = re.split(r"\n\s*Function : ", full)
    sass = "\n".join(p for p in parts if p.startswith("_ZN3tfn16tfn_strip_kernel"))
    assert sass
    # the fp64 gradient path and the MUFU reciprocals are in the strip kernel
    for op in ("DFMA", "MUFU.RCP64H", "MUFU.RCP", "LDG.E.128", "STG.E"):
        assert op in sass, op


def test_status_strings_and_version(so):
    from paper_2005_08165_b200 import tfn
    assert tfn.tfn_status_string(0) == "TFN_OK"
    assert tfn.tfn_status_string(2) == "TFN_ERR_CONFIG"
    assert tfn.tfn_version() >= 100


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_gpu_fails_loudly(so):
    from paper_2005_08165_b200 import Estimator, TfnError
    with pytest.raises(TfnError) as e:
        Estimator((500, 500, 320, 240))
    assert e.value.status == 3      # TFN_ERR_CUDA: no silent CPU path


def test_create_rejects_bad_config_before_touching_the_device(so):
    from paper_2005_08165_b200 import tfn
    with pytest.raises(tfn.TfnError) as e:
        tfn.tfn_create((0.0, 500, 320, 240), 1, 1)
    assert e.value.status == 2
    with pytest.raises(tfn.TfnError) as e:
        tfn.tfn_create((float("nan"), 500, 320, 240), 1, 1)
    assert e.value.status == 2
    with pytest.raises(tfn.TfnError) as e:
        tfn.tfn_create((500, 500, 320, 240), 7, 1)
    assert e.value.status == 1


def test_oracle_and_product_share_no_code():
    """The product package never imports/includes oracle/, and the oracle never
    imports/includes the product (comments may name each other)."""
    imp = re.compile(r"^\s*(?:import|from)\s+(\S+)|^\s*#\s*include\s*[<\"]([^>\"]+)", re.M)
    prod = os.path.join(ROOT, "paper_2005_08165_b200")
    for dirpath, _, files in os.walk(prod):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                for a, b in imp.findall(open(os.path.join(dirpath, f)).read()):
                    assert "oracle" not in (a or b), (f, a or b)
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c")):
            for a, b in imp.findall(open(os.path.join(ROOT, "oracle", f)).read()):
                t = a or b
                assert "paper_2005" not in t and "tfn_" not in t and "tfn_scenes" not in t, (f, t)


def test_auto_state_machine_host_logic(so):
    """AUTO (tfn_abi.cu) without a device: fast -> masked -> general above 20 % of probed row
    steps needing the special path, back below 10 %; probe schedule: fast / masked count every
    8th call, masked re-probes fast every 256th call, general re-probes masked every 32nd;
    nothing is probed (or re-probed) when no read-back is possible (CUDA-graph capture)."""
    from paper_2005_08165_b200 import tfn as T
    nxt = lambda st, pv, r: T.tfn_debug_auto(st, pv, r, 1, False)[0]  # noqa: E731
    # transitions after a fast probe
    assert nxt(0, 0, 0.5) == 1 and nxt(0, 0, 0.15) == 0 and nxt(0, 0, 0.01) == 0
    assert nxt(1, 0, 0.5) == 1 and nxt(1, 0, 0.05) == 0 and nxt(2, 0, 0.05) == 0 and nxt(2, 0, 0.5) == 2
    # transitions after a masked probe
    assert nxt(1, 1, 0.5) == 2 and nxt(1, 1, 0.05) == 1 and nxt(1, 1, 0.15) == 1
    assert nxt(2, 1, 0.05) == 1 and nxt(2, 1, 0.15) == 2 and nxt(2, 1, 0.5) == 2
    pick = lambda st, n, cp=True: T.tfn_debug_auto(st, 0, 0.0, n, cp)[1:]  # noqa: E731
    assert pick(0, 0) == (0, True) and pick(0, 3) == (0, False) and pick(0, 8) == (0, True)
    assert pick(0, 8, False) == (0, False)
    assert pick(1, 256) == (0, True) and pick(1, 8) == (1, True) and pick(1, 5) == (1, False)
    assert pick(1, 256, False) == (1, False)                  # capture: no re-probe
    assert pick(2, 32) == (1, True) and pick(2, 8) == (2, False) and pick(2, 32, False) == (2, False)
    with pytest.raises(T.TfnError):
        T.tfn_debug_auto(3, 0, 0.0, 0, True)
