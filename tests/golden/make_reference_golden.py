"""Generate golden fixtures by importing the reference (lorasched) itself.

Run in the build container (the reference is not present on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_reference_golden.py

Writes
  traffic_reference.json   lorasched.costmodel.traffic() per-kernel bytes for every variant
                           and pass at the BASELINE configs plus assorted shapes, the frozen
                           totals of pkg/tests/test_costmodel.py:22-27, and the
                           POST /v1/traffic response of pkg/tests/test_service.py:140-150.
  schedule_reference.json  a lorasched schedule document (ls/schedule.py:441-490) planned for
                           pkg/tests/conftest.py's mixed_workload(4) at capacity 8192,
                           stage_count 1 — the real producer of FusedMultiLoRA segment tables.
"""
from __future__ import annotations

import json
import os
import sys
import warnings

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, REF_TESTS)
    from lorasched import costmodel as cm

    shapes = [
        (8192, 4096, 4096, 16, 2),  # reference test shape
        (8192, 4096, 4096, 0, 2),
        (2048, 4096, 4096, 16, 2),  # C1
        (8192, 4096, 1024, 16, 2),  # C2 k/v
        (8192, 4096, 14336, 16, 2),  # C2 gate/up
        (8192, 14336, 4096, 16, 2),  # C2 down
        (16384, 8192, 8192, 16, 2),  # C4 q/o
        (16384, 8192, 28672, 16, 2),  # C4 gate/up
        (16384, 28672, 8192, 16, 2),  # C4 down
        (8192, 4096, 4096, 64, 2),
        (8192, 4096, 4096, 8, 1),
        (130, 72, 200, 8, 4),
        (1, 1, 1, 1, 2),
        (129, 256, 8, 32, 2),
    ]
    rows = []
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for m, k, n, r, e in shapes:
            shape = cm.GemmShape(m=m, k=k, n=n, r=r, element_bytes=e)
            for variant in cm.VARIANTS:
                for p in cm.PASSES:
                    rep = cm.traffic(shape, p, variant)
                    rows.append({"shape": [m, k, n, r, e], "variant": variant, "pass": p, "report": rep.to_dict()})
    doc = {
        "generator": "lorasched.costmodel (reference) via tests/golden/make_reference_golden.py",
        "frozen_totals": {  # pkg/tests/test_costmodel.py:22-27
            "REF_FROZEN_TOTAL": 503_316_480,
            "REF_UNFUSED_TOTAL": 1_344_536_576,
            "REF_FUSED_TOTAL": 807_403_520,
        },
        "eq2_reference": cm.arithmetic_intensity(16, 4096, 8192),
        "memory_reference": cm.lora_memory_bytes(4096, 4096, 16).to_dict(),
        "reports": rows,
    }
    try:
        from fastapi.testclient import TestClient
        from lorasched.service.app import create_app

        client = TestClient(create_app())
        resp = client.post("/v1/traffic", json={"m": 8192, "k": 4096, "n": 4096, "r": 16, "variant": "unfused"})
        doc["service_traffic_unfused"] = resp.json()
        resp = client.post("/v1/traffic", json={"m": 8192, "k": 4096, "n": 4096, "r": 16, "variant": "fused_multi_lora"})
        doc["service_traffic_multi"] = resp.json()
    except Exception as exc:  # pragma: no cover - optional dependency path
        doc["service_error"] = repr(exc)
    with open(os.path.join(HERE, "traffic_reference.json"), "w") as f:
        json.dump(doc, f, indent=1, sort_keys=True)

    # schedule document from the real planner
    from conftest import mixed_workload  # reference tests' workload builder
    from lorasched.packing import SolverBudget
    from lorasched.planner import plan_schedule
    from lorasched.schedule import schedule_to_doc

    specs, samples = mixed_workload(4, samples_per_adapter=32, global_batch_size=8, padding_multiple=64)
    plan = plan_schedule(specs, samples, capacity=8192, budget=SolverBudget(timeout_s=2.0, node_limit=20000), group_size=4,
                         stage_count=1)
    sdoc = schedule_to_doc(plan.schedule, specs)
    with open(os.path.join(HERE, "schedule_reference.json"), "w") as f:
        json.dump(sdoc, f, indent=1, sort_keys=True)
    print("wrote", len(rows), "traffic reports and", len(sdoc["entries"]), "schedule entries")


if __name__ == "__main__":
    main()
