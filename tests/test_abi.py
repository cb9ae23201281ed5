"""CPU-side checks of the boundary (-m "not gpu"): the C-ABI library loads, exports every
symbol include/bpt.h declares, and fails loudly (no CPU fallback) without a GPU."""
import ctypes
import os
import re
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_declares_the_boundary():
    import paper_2311_10201_b200 as bpt
    syms = bpt.header_symbols()
    for name in ["bpt_graph_load", "bpt_sample", "bpt_select_seeds", "bpt_rrr_extract", "bpt_rrr_sizes",
                 "bpt_rrr_digests", "bpt_comm_init", "bpt_last_error"]:
        assert name in syms


def test_library_exports_every_header_symbol():
    import paper_2311_10201_b200 as bpt
    lib = ctypes.CDLL(bpt.LIB_PATH)
    missing = [s for s in bpt.header_symbols() if not hasattr(lib, s)]
    assert missing == []
    out = subprocess.run(["nm", "-D", "--defined-only", bpt.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (bpt_[a-z_0-9]+)", out))
    assert set(bpt.header_symbols()) <= exported
    assert bpt.bpt_abi_version() == 2


def test_header_constants_match_binding():
    """Every #define / enum value of include/bpt.h that the binding mirrors has the same value."""
    import paper_2311_10201_b200 as bpt
    hdr = open(os.path.join(ROOT, "include", "bpt.h")).read()
    defs = {k: int(v.rstrip("u"), 0) for k, v in re.findall(r"#define (BPT_FLAG_[A-Z_]+) (\w+)", hdr)}
    assert defs == {f"BPT_{name}": getattr(bpt, name) for name in
                    ("FLAG_PROFILE", "FLAG_WIDE", "FLAG_SPARSE", "FLAG_LT_FUSED", "FLAG_LT_DENSE", "FLAG_LT_REWALK",
                     "FLAG_LT_LEVELS", "FLAG_QUEUE", "FLAG_UNSORTED", "FLAG_PULL", "FLAG_SLOTWISE")}
    flags = list(defs.values())
    assert len(set(flags)) == len(flags) and all(f & (f - 1) == 0 for f in flags)  # distinct single bits
    enums = dict((k, int(v)) for k, v in re.findall(r"(BPT_E[A-Z]+|BPT_OK)\s*=\s*(-?\d+)", hdr))
    for k in ("BPT_OK", "BPT_EINVAL", "BPT_ENOMEM", "BPT_ECUDA", "BPT_ENCCL", "BPT_ESTATE"):
        assert enums[k] == getattr(bpt, k)
    assert dict(re.findall(r"(BPT_IC|BPT_LT)\s*=\s*(\d+)", hdr)) == {"BPT_IC": str(bpt.IC), "BPT_LT": str(bpt.LT)}


def test_import_before_torch():
    """Loading libbpt.so before torch must not pin an older NCCL under the shared soname
    (torch's libtorch_cuda needs the NCCL it was built with)."""
    r = subprocess.run([sys.executable, "-c", "import paper_2311_10201_b200, torch; print('ok')"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_library_is_sm100a_cuda():
    import paper_2311_10201_b200 as bpt
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", bpt.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_oracle_in_product():
    """The product never imports / links the oracle (DESIGN.md §Oracle independence)."""
    pkg = os.path.join(ROOT, "paper_2311_10201_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "import oracle" not in text and "oracle.c" not in text and "_oracle.so" not in text, f
    import paper_2311_10201_b200 as bpt
    out = subprocess.run(["ldd", bpt.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in out


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="checks the no-GPU failure path")
def test_fails_loudly_without_gpu():
    import paper_2311_10201_b200 as bpt
    with pytest.raises(bpt.BptError) as ei:
        bpt.Graph(np.array([0, 1], dtype=np.uint64), np.array([0], dtype=np.uint32),
                  w_q31=np.array([5], dtype=np.uint32))
    assert ei.value.code == bpt.BPT_ECUDA
