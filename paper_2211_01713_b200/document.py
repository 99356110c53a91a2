"""Plan documents: the wire format every reference comparison uses.

Host serialization of a ``Plan`` into the reference's JSON document
(``problem.py:290-341``), the inverse used by ``predict``/``simulate``
(``problem.py:344-361``), and the atomic writer (``problem.py:384-398``).
The predictions inside a document come from the device ``_build_plan``
(``k_place`` predict phase or ``k_eval_states``); nothing here computes
model values.
"""

from __future__ import annotations

import json
import os
import tempfile
from pathlib import Path
from typing import Any, Mapping

from .errors import ProblemFormatError
from .layout import ROW_FIELDS
from .model import Allocation, slo_check


def _breakdown_dict(bd) -> dict[str, float]:
    return {f: getattr(bd, f) for f in ROW_FIELDS}


def plan_to_document(plan, specs: Mapping[str, Any]) -> dict[str, Any]:
    """Serialize a plan with its predictions and per-workload SLO checks."""
    gpus = []
    for gpu in plan.gpus:
        allocations = []
        for alloc in gpu.allocations:
            bd = gpu.predicted[alloc.workload]
            check = slo_check(bd, specs[alloc.workload])
            allocations.append({
                "workload": alloc.workload,
                "r": alloc.r,
                "batch": alloc.batch,
                "predicted": _breakdown_dict(bd),
                "slo": {"latency_ok": check.latency_ok, "throughput_ok": check.throughput_ok},
            })
        gpus.append({"gpu_index": gpu.gpu_index, "fragment_r": gpu.fragment_r,
                     "allocations": allocations})
    return {
        "strategy": plan.strategy,
        "gpu_type": plan.gpu_type,
        "cost_per_hour": plan.cost_per_hour,
        "gpus": gpus,
        "diagnostics": list(plan.diagnostics),
        "per_workload_r_inter": dict(sorted(plan.per_workload_r_inter.items())),
    }


def _field(mapping: Mapping[str, Any], key: str, context: str) -> Any:
    if key not in mapping:
        raise ProblemFormatError(f"{context}: missing required field {key!r}")
    return mapping[key]


def allocations_from_document(doc: Mapping[str, Any], context: str = "plan") -> list[list[Allocation]]:
    """Per-device allocations of a plan document (predictions are ignored)."""
    out = []
    for i, gpu in enumerate(_field(doc, "gpus", context)):
        out.append([
            Allocation(workload=str(_field(raw, "workload", context)),
                       r=float(_field(raw, "r", context)),
                       batch=int(_field(raw, "batch", context)))
            for raw in _field(gpu, "allocations", f"{context}: gpus[{i}]")
        ])
    return out


def write_json_atomic(path, doc: Mapping[str, Any]) -> None:
    """Write via a temporary file and rename, so readers never see a partial file."""
    path = Path(path)
    path.parent.mkdir(parents=True, exist_ok=True)
    fd, tmp = tempfile.mkstemp(dir=path.parent, suffix=".tmp")
    try:
        with os.fdopen(fd, "w") as handle:
            json.dump(doc, handle, indent=2)
            handle.write("\n")
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise
