"""CPU: the C-ABI library loads and exports every symbol include/psb.h declares."""
import os
import re
import subprocess

from tests.conftest import ROOT


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "psb.h")).read()
    return sorted(set(re.findall(r"^PSB_API [^(]*?\b(psb_\w+)\(", src, flags=re.M)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("psb_ctx_create", "psb_ef_topk", "psb_sparse_mean_sgd", "psb_sync_step",
              "psb_async_round", "psb_q8_quantize", "psb_ef_onebit"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2506_17551_b200 import _lib
    lib = _lib.load()
    assert lib.psb_abi_version() == 1
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (psb_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    # and the Python binding covers all of them
    assert set(_lib.EXPORTED) == set(declared_symbols())


def test_library_is_sm100a_only():
    from paper_2506_17551_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_payload_sizes():
    from paper_2506_17551_b200 import _lib
    lib = _lib.load()
    assert lib.psb_status_string(_lib.PSB_ENONFINITE) == b"non-finite entry"
    # TOPK f32: u32 idx[k] | pad16 | f32 val[k] | pad16
    assert lib.psb_payload_bytes(_lib.PSB_COMP_TOPK, _lib.PSB_F32, 10) == 48 + 48
    assert lib.psb_payload_bytes(_lib.PSB_COMP_TOPK, _lib.PSB_F64, 4) == 16 + 32
    assert lib.psb_payload_bytes(_lib.PSB_COMP_TOPK_Q8, _lib.PSB_F32, 130) == 528 + 144 + 16


def test_no_cuda_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        return
    from paper_2506_17551_b200 import PsbError
    from paper_2506_17551_b200.engine import Context
    try:
        Context(1024)
    except PsbError:
        return
    raise AssertionError("Context() without a GPU must raise, not fall back")
