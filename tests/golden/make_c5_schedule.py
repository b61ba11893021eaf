"""Generate the C5 schedule fixture by running the reference's own planner.

BASELINE.json configs[4]: "LLaMa-3.1-8B 4 concurrent LoRA jobs, full decoder fwd+bwd step,
bin-packed microbatches on 8xB200 with dA/dB allreduce". The four jobs are
pkg/tests/conftest.py's ``mixed_workload(4)`` length profiles (SHORT / MEDIUM / LONG /
MIXED) with the C3 adapter hyper-parameters: lora_rank 8/16/32/64,
alpha = 2·rank (scaling 2.0), dropout 0/0.05/0.1/0.1, padding multiple 64, global batch 8.
lorasched's ``plan_schedule`` (ls/planner.py:23-118) packs them at capacity 8192 with one
pipeline stage (S = 1, the DP setting of SURVEY.md §8(e)); ``schedule_to_doc``
(ls/schedule.py:441-490) serialises the plan. The document is what an external training
system consumes (reference SPEC.md:386) and what ``bench.py --config c5`` and
``paper_2510_00206_b200.decoder`` read — /root/reference is not needed at run time.

    python tests/golden/make_c5_schedule.py     # needs /root/reference (this container)
"""
from __future__ import annotations

import dataclasses
import json
import os
import sys

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))

RANKS = (8, 16, 32, 64)
DROPOUT = (0.0, 0.05, 0.1, 0.1)


def main() -> None:
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, REF_TESTS)
    from conftest import mixed_workload  # reference tests' workload builder
    from lorasched.packing import SolverBudget
    from lorasched.planner import plan_schedule
    from lorasched.schedule import schedule_to_doc

    specs, samples = mixed_workload(4, samples_per_adapter=64, global_batch_size=8, padding_multiple=64)
    specs = [dataclasses.replace(s, lora_rank=r, alpha=2.0 * r, dropout_p=p)
             for s, r, p in zip(specs, RANKS, DROPOUT)]
    plan = plan_schedule(specs, samples, capacity=8192, budget=SolverBudget(timeout_s=2.0, node_limit=20000),
                         group_size=4, stage_count=1)
    doc = schedule_to_doc(plan.schedule, specs)
    with open(os.path.join(HERE, "schedule_c5.json"), "w") as f:
        json.dump(doc, f, indent=1, sort_keys=True)
    tot = [e.get("total_padded_tokens") for e in doc["entries"] if e["kind"] == "microbatch"]
    print("wrote", len(tot), "microbatches; padded tokens", tot)


if __name__ == "__main__":
    main()
