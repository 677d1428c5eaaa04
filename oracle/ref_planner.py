"""TEST INFRASTRUCTURE ONLY — the reference planner itself, as the plan-parity checker.

oracle/_ref/libparplan_ref.so is built by oracle/Makefile directly from the reference's own
sources (/root/reference/proj/src/{model_ir,cluster,strategy,cost_model,planner,oracle}.cc,
namespace renamed to parplan_ref) plus this repo's C surface compiled with the ref_plan_
prefix.  Plan parity is therefore pinned against the reference's actual code, not a
restatement.  The library is built here (where /root/reference exists) and travels to the
GPU box as a prebuilt file.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libparplan_ref.so")

_api = None


def available() -> bool:
    return os.path.exists(REF_LIB)


def api():
    global _api
    if _api is None:
        from paper_2211_13878_b200 import _lib
        from paper_2211_13878_b200.planner import PlanAPI
        if not available():
            raise ImportError(f"{REF_LIB} missing: run `make -C oracle` where /root/reference exists")
        L = ctypes.CDLL(REF_LIB)
        _lib.declare_plan_api(L, "ref_plan_")
        _api = PlanAPI(L, "ref_plan_")
    return _api
