"""The C-ABI libraries load and export every symbol include/eps_capi.h declares.

CPU only: symbols are resolved, nothing is called that needs a GPU.
"""
import ctypes
import os
import re

import pytest

from paper_2102_03161_b200 import LIB_PATH

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include/eps_capi.h")
REF_LIB = os.path.join(ROOT, "oracle/_ref/libeps_ref.so")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    shared, product = src.split("#ifndef EPS_REFERENCE_BUILD", 1)
    common = sorted(set(re.findall(r"EPS_FN\((\w+)\)\s*\(", shared)))
    extra = sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(eps_\w+)\s*\(", product, flags=re.M)))
    return common, extra


def test_header_parses():
    common, extra = declared()
    assert "next_frozen_count" in common and "load_balance" in common
    assert "eps_gemm_bf16" in extra and "eps_vit_train_step" in extra


def test_product_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB_PATH)
    common, extra = declared()
    missing = [n for n in ["eps_" + c for c in common] + extra if not hasattr(lib, n)]
    assert not missing, missing


def test_reference_build_exports_control_plane():
    if not os.path.exists(REF_LIB):
        pytest.skip("oracle/_ref not built (make oracle)")
    lib = ctypes.CDLL(REF_LIB)
    common, _ = declared()
    missing = [n for n in ["epsref_" + c for c in common] if not hasattr(lib, n)]
    assert not missing, missing
