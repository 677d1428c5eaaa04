"""Python mirror of the reference plan/search interface over the gx_plan_* C ABI.

Reference interface (proj/include/parplan/planner.h, cost_model.h, strategy.h, oracle.h):
``Optimize``, ``ExhaustivePlan``, ``DpSearch``, ``ExhaustiveDp``, ``EstimateLayerCost`` /
``EstimateMemory``, ``TransformationCostMs``, ``EnumerateStrategies``,
``PartitionPipeline``, ``StagePipelineCostMs``, ``CollectiveVolumeBytes``,
``GroupBandwidthGbps``.  Errors keep the reference's behaviour: invalid inputs raise
``ValidationError``, oracle guard trips raise ``GuardError``, and infeasibility is a value
(``PlanOutcome.plan is None`` with the diagnostic), never an exception.

`PlanAPI` is parameterised by library + symbol prefix so the test-only checker
(oracle/ref_planner.py, prefix ``ref_plan_``) exposes exactly the same surface.
"""
from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass
from typing import Any, Optional, Sequence

from . import _lib

_KINDS = {"all_reduce": 0, "all_gather": 1, "reduce_scatter": 2}


def _text(obj) -> bytes:
    if obj is None:
        return None
    if isinstance(obj, (bytes, bytearray)):
        return bytes(obj)
    if isinstance(obj, str):
        return obj.encode()
    return json.dumps(obj).encode()


@dataclass
class PlanOutcome:
    """parplan::PlanOutcome (planner.h:132-137): plan JSON (PlanToJson) or diagnostic."""
    plan: Optional[dict]
    plan_text: Optional[str]
    diagnostic: str

    def feasible(self) -> bool:
        return self.plan is not None


class PlanAPI:
    def __init__(self, lib: ctypes.CDLL, prefix: str):
        self._L = lib
        self._p = prefix

    def _fn(self, name):
        return getattr(self._L, self._p + name)

    def _err(self) -> str:
        return self._fn("last_error")().decode()

    def _raise(self, code: int):
        msg = self._err()
        if code == 5:
            raise _lib.GuardError(code, msg)
        raise _lib.ValidationError(code, msg)

    _BUF = 1 << 20  # plan JSON of a 96-layer model is ~40 KB: one call nearly always fits

    def _call_text(self, name, *args) -> tuple[int, str]:
        """One C call into a generously sized buffer (the search runs once); only an output
        longer than the buffer costs a second call with the exact size."""
        needed = ctypes.c_size_t(0)
        buf = ctypes.create_string_buffer(self._BUF)
        code = self._fn(name)(*args, buf, self._BUF, ctypes.byref(needed))
        if code not in (0, 2) and needed.value > self._BUF:
            buf = ctypes.create_string_buffer(needed.value)
            code = self._fn(name)(*args, buf, needed.value, ctypes.byref(needed))
        if code not in (0, 2):
            self._raise(code)
        return code, buf.value.decode()

    @staticmethod
    def _batches(batches):
        if not batches:
            return None, 0
        arr = (ctypes.c_int * len(batches))(*batches)
        return arr, len(batches)

    # ------------------------------------------------------------------ search
    def optimize(self, model, cluster, profile=None, batches: Sequence[int] = None,
                 prune=True, guideline="layers", num_threads=1) -> PlanOutcome:
        arr, n = self._batches(batches)
        code, text = self._call_text("optimize", _text(model), _text(cluster), _text(profile),
                                     arr, n, int(prune), guideline.encode(), int(num_threads))
        if code == 2:
            return PlanOutcome(None, None, text)
        return PlanOutcome(json.loads(text), text, "")

    def exhaustive_plan(self, model, cluster, profile=None, batches: Sequence[int] = None,
                        prune=True, guideline="layers") -> PlanOutcome:
        arr, n = self._batches(batches)
        code, text = self._call_text("exhaustive", _text(model), _text(cluster), _text(profile),
                                     arr, n, int(prune), guideline.encode())
        if code == 2:
            return PlanOutcome(None, None, text)
        return PlanOutcome(json.loads(text), text, "")

    def dp_search(self, model, begin, end, budget_bytes, group_size, batch, bandwidth_gbps,
                  profile=None, prune=True, exhaustive=False) -> dict:
        _, text = self._call_text("exhaustive_dp" if exhaustive else "dp_search", _text(model),
                                  int(begin), int(end), int(budget_bytes), int(group_size),
                                  int(prune), int(batch), float(bandwidth_gbps), _text(profile))
        out = json.loads(text)
        out["_text"] = text
        return out

    # --------------------------------------------------------------- cost model
    def estimate(self, param_bytes, act_bytes, fwd_ms, strategy, batch, bandwidth_gbps,
                 profile=None) -> dict:
        _, text = self._call_text("estimate", int(param_bytes), int(act_bytes), float(fwd_ms),
                                  strategy.encode(), int(batch), float(bandwidth_gbps),
                                  _text(profile))
        out = json.loads(text)
        out["_text"] = text
        return out

    def transformation_ms(self, param_bytes, act_bytes, prev, cur, batch, bandwidth_gbps) -> float:
        v = ctypes.c_double(0)
        code = self._fn("transformation_ms")(int(param_bytes), int(act_bytes), prev.encode(),
                                             cur.encode(), int(batch), float(bandwidth_gbps),
                                             ctypes.byref(v))
        if code:
            self._raise(code)
        return v.value

    def collective_bytes(self, kind: str, degree: int, payload: float) -> float:
        v = ctypes.c_double(0)
        code = self._fn("collective_bytes")(_KINDS[kind], int(degree), float(payload),
                                            ctypes.byref(v))
        if code:
            self._raise(code)
        return v.value

    def pipeline_cost(self, stage_costs: Sequence[float], pp_degree: int, micro_batches: int) -> float:
        arr = (ctypes.c_double * len(stage_costs))(*stage_costs)
        v = ctypes.c_double(0)
        code = self._fn("pipeline_cost")(arr, len(stage_costs), int(pp_degree), int(micro_batches),
                                         ctypes.byref(v))
        if code:
            self._raise(code)
        return v.value

    # -------------------------------------------------------- strategies / misc
    def enumerate(self, group_size: int, prune: bool) -> dict:
        _, text = self._call_text("enumerate", int(group_size), int(prune))
        return json.loads(text)

    def partition(self, model, pp_degree: int, guideline="layers") -> Optional[list]:
        _, text = self._call_text("partition", _text(model), int(pp_degree), guideline.encode())
        return json.loads(text)

    def validate(self, kind: str, obj) -> None:
        code = self._fn("validate")(kind.encode(), _text(obj))
        if code:
            self._raise(code)

    def bandwidth(self, cluster, group_size: int) -> float:
        v = ctypes.c_double(0)
        code = self._fn("bandwidth")(_text(cluster), int(group_size), ctypes.byref(v))
        if code:
            self._raise(code)
        return v.value


_api: Optional[PlanAPI] = None


def api() -> PlanAPI:
    """The product planner (libgx.so, namespace parplan written in this repo)."""
    global _api
    if _api is None:
        _api = PlanAPI(_lib.lib(), "gx_plan_")
    return _api


def ribbon(plan: dict) -> str:
    """Run-length per-layer strategy summary, e.g. "[dp:8] x6 | [sdp:8] x26" (the format of
    the reference CLI summary, proj/tools/parplan_main.cc:95-111)."""
    parts = []
    for st in plan["stages"]:
        runs: list[list[Any]] = []
        for layer in st["layers"]:
            s = layer["strategy"] or "serial"
            if runs and runs[-1][0] == s:
                runs[-1][1] += 1
            else:
                runs.append([s, 1])
        parts.append(" | ".join(f"[{s}] x{n}" for s, n in runs))
    return " || ".join(parts)
