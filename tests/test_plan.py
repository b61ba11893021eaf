"""Host-side segment tables, routing and schedule ingestion (no GPU)."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest
import torch

from oracle import routing as orouting
from paper_2510_00206_b200 import AdapterConfig, LayerPlan, Segment, padded_rank, segments_from_lengths
from paper_2510_00206_b200 import schedule as sched
from paper_2510_00206_b200.errors import ValidationError
from paper_2510_00206_b200.plan import split_segments, validate_segments

GOLD_SCHED = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "schedule_reference.json")))


def test_padded_rank():
    assert [padded_rank(r) for r in (1, 8, 16, 17, 32, 64)] == [16, 16, 16, 32, 32, 64]


def test_adapter_config_validation():
    with pytest.raises(ValidationError):
        AdapterConfig(rank=0)
    with pytest.raises(ValidationError):
        AdapterConfig(rank=8, dropout_p=1.0)
    with pytest.raises(ValidationError):
        AdapterConfig(rank=8, scaling=float("inf"))

    class Spec:  # lorasched AdapterSpec fields (ls/workload.py:25-48)
        lora_rank, alpha, dropout_p = 16, 32.0, 0.05

    c = AdapterConfig.from_adapter_spec(Spec(), seed=3)
    assert (c.rank, c.scaling, c.dropout_p, c.seed) == (16, 2.0, 0.05, 3)


def test_plan_columns_and_problem():
    ads = [AdapterConfig(8, 2.0, 0.0, 1), AdapterConfig(16, 1.0, 0.1, 2), AdapterConfig(64, 0.5, 0.1, 3)]
    segs = segments_from_lengths([0, 1, 2, 1], [100, 200, 300, 50], batches=[0, 0, 0, 1])
    # default: one column block per adapter (segments 1 and 3 = adapter 1 share it)
    shared = LayerPlan(700, 256, 128, ads, segs, offset=5)
    assert shared.col_starts == [0, 16, 32, 16] and shared.rank_total == 96
    assert shared.adapter_grad_slices() == [(0, 0, 8), (1, 16, 16), (2, 32, 64)]
    assert shared.column_blocks() == [(0, 0, 16), (1, 16, 16), (2, 32, 64)]
    a_cat = shared.gather_a([torch.full((r.rank, 256), float(i + 1)) for i, r in enumerate(ads)])
    b_cat = shared.gather_b([torch.full((128, r.rank), float(i + 1)) for i, r in enumerate(ads)])
    assert a_cat.shape == (96, 256) and b_cat.shape == (128, 96)
    assert a_cat[:8].eq(1).all() and a_cat[8:16].eq(0).all() and a_cat[16:32].eq(2).all() and a_cat[32:].eq(3).all()
    assert b_cat[:, 16:32].eq(2).all() and b_cat[:, 8:16].eq(0).all()
    assert shared.host_routes()[5] == (3, 3, 16, 32)  # rows 640..699: segment 3 only
    assert shared.host_routes()[4] == (2, 3, 16, 96)  # segments 2|3: hull of blocks [32,96) and [16,32)
    assert shared.host_routes()[2] == (1, 2, 16, 96)  # rows 256..383 straddle segments 1|2
    # per-(adapter, batch) slots: one block per segment
    plan = LayerPlan(700, 256, 128, ads, segs, offset=5, share_blocks=False)
    assert plan.ranks == [16, 16, 64, 16]
    assert plan.col_starts == [0, 16, 32, 96]
    assert plan.rank_total == 112
    p = plan.problem
    assert p.num_segments == 4 and p.rank_total == 112
    assert (p.segments[2].row_start, p.segments[2].row_end, p.segments[2].col_start, p.segments[2].rank) == (300, 600,
                                                                                                           32, 64)
    assert p.segments[1].seed == 2 and p.segments[3].offset == 5
    assert plan.needs_keep_bits
    assert plan.segment_grad_slices() == [(0, 0, 0, 8), (1, 0, 16, 16), (2, 0, 32, 64), (1, 1, 96, 16)]
    # eval mode: no dropout anywhere
    ev = LayerPlan(700, 256, 128, ads, segs, training=False)
    assert not ev.needs_keep_bits and all(ev.problem.segments[i].dropout_p == 0 for i in range(4))


def test_shared_blocks_non_adjacent_routes_hull():
    """a0, a1, a0: the third segment reuses block 0, so a tile straddling a1|a0 spans the
    hull [0, 32) — the device table (lf_build_routes) and the oracle agree on it."""
    ads = [AdapterConfig(16), AdapterConfig(8)]
    segs = [Segment(0, 0, 200), Segment(1, 200, 392), Segment(0, 392, 640, 1)]
    plan = LayerPlan(640, 64, 64, ads, segs)
    assert plan.col_starts == [0, 16, 0] and plan.rank_total == 32
    ref = orouting.routes([(s.row_start, s.row_end) for s in segs], list(zip(plan.col_starts, plan.ranks)), 640)
    assert np.array_equal(np.array(plan.host_routes(), np.int32), ref)
    assert tuple(ref[3]) == (1, 2, 0, 32)  # rows 384..511
    assert orouting.column_blocks([16, 8, 16], adapters=[0, 1, 0]) == [0, 16, 0]


def test_plan_rejects_bad_tables():
    ads = [AdapterConfig(16)]
    with pytest.raises(ValidationError):
        LayerPlan(100, 64, 64, ads, [Segment(0, 0, 120)])
    with pytest.raises(ValidationError):
        LayerPlan(100, 64, 64, ads, [Segment(1, 0, 50)])
    with pytest.raises(ValidationError):
        LayerPlan(100, 64, 64, ads, [Segment(0, 50, 100), Segment(0, 0, 50)])
    with pytest.raises(ValidationError):  # R > 128
        LayerPlan(300, 64, 64, [AdapterConfig(64)] * 3, segments_from_lengths([0, 1, 2], [100, 100, 100]))
    with pytest.raises(ValidationError):
        LayerPlan(64, 64, 64, ads * 33, segments_from_lengths(list(range(33)), [1] * 33))


@pytest.mark.parametrize("lengths", [(3584, 2432, 1408, 768), (3520, 2496, 1408, 768), (100, 0, 5, 300)])
def test_host_routes_match_oracle(lengths):
    ads = [AdapterConfig(r) for r in (8, 16, 32, 64)]
    segs = segments_from_lengths([0, 1, 2, 3], lengths)
    m = sum(lengths) + 77
    plan = LayerPlan(m, 64, 64, ads, segs)
    ref = orouting.routes([(s.row_start, s.row_end) for s in segs], list(zip(plan.col_starts, plan.ranks)), m)
    assert np.array_equal(np.array(plan.host_routes(), np.int32), ref)
    assert len(plan.host_routes()) * orouting.ENTRY_BYTES == orouting.table_bytes(m)


def test_straddling_tiles_with_p64():
    """P = 64 padding (ls/workload.py:31) puts two segments in one 128-row tile."""
    segs = segments_from_lengths([0, 1, 2, 3], [3520, 2496, 1408, 768])
    plan = LayerPlan(8192, 64, 64, [AdapterConfig(r) for r in (8, 16, 32, 64)], segs)
    routes = plan.host_routes()
    straddle = [t for t, r in enumerate(routes) if r[1] > r[0]]
    assert straddle == [27]  # rows 3456..3583 hold segments 0 and 1
    assert routes[27] == (0, 1, 0, 32)


def test_schedule_document_ingestion():
    """A real lorasched schedule (tests/golden/schedule_reference.json, produced by the
    reference planner) becomes segment tables whose padded lengths match the document."""
    ids, cfgs = sched.adapters_from_doc(GOLD_SCHED)
    assert ids == [a["adapter_id"] for a in GOLD_SCHED["adapters"]]
    assert all(c.scaling == a["alpha"] / a["lora_rank"] for c, a in zip(cfgs, GOLD_SCHED["adapters"]))
    mbs = sched.microbatches_from_doc(GOLD_SCHED)
    entries = [e for e in GOLD_SCHED["entries"] if e["kind"] == "microbatch"]
    assert len(mbs) == len(entries)
    for mb, e in zip(mbs, entries):
        assert mb.rows == e["total_padded_tokens"] <= GOLD_SCHED["capacity"]
        assert mb.raw_tokens == e["total_raw_tokens"]
        assert [s.rows for s in mb.segments] == [s["padded_tokens"] for s in e["segments"]]
        assert [s.batch for s in mb.segments] == [s["global_batch_index"] for s in e["segments"]]
        assert [ids[s.adapter] for s in mb.segments] == [s["adapter_id"] for s in e["segments"]]
        # packed sequences: every sample, then the segment's pad rows as one pseudo-sequence
        want = []
        for s in e["segments"]:
            want += [r["length"] for r in s["samples"]]
            if s["padded_tokens"] > s["raw_tokens"]:
                want.append(s["padded_tokens"] - s["raw_tokens"])
        assert list(mb.sequences) == want and sum(mb.sequences) == mb.rows
        plan = LayerPlan(mb.rows, 4096, 4096, cfgs, list(mb.segments))
        ref = orouting.routes([(s.row_start, s.row_end) for s in mb.segments],
                              list(zip(plan.col_starts, plan.ranks)), mb.rows)
        assert np.array_equal(np.array(plan.host_routes(), np.int32), ref)


def test_schedule_validation():
    bad = json.loads(json.dumps(GOLD_SCHED))
    bad["schema_version"] = 2
    with pytest.raises(ValidationError, match="schema_version"):
        sched.microbatches_from_doc(bad)
    bad = json.loads(json.dumps(GOLD_SCHED))
    bad["entries"][0]["segments"][0]["padded_tokens"] += 64
    with pytest.raises(ValidationError, match="padded_tokens"):
        sched.microbatches_from_doc(bad)
    bad = json.loads(json.dumps(GOLD_SCHED))
    bad["entries"][0]["segments"][0]["adapter_id"] = "nope"
    with pytest.raises(ValidationError, match="unknown adapter"):
        sched.microbatches_from_doc(bad)
    bad = json.loads(json.dumps(GOLD_SCHED))
    del bad["entries"][0]["group_id"]
    with pytest.raises(ValidationError, match="group_id"):
        sched.microbatches_from_doc(bad)


def test_segments_from_microbatch_objects():
    class Seg:
        def __init__(self, a, b, n):
            self.adapter_id, self.global_batch_index, self.padded_tokens = a, b, n

    class MB:
        segments = (Seg("a0", 3, 128), Seg("a2", 3, 64), Seg("a2", 4, 192))

    segs = sched.segments_from_microbatch(MB(), ["a0", "a1", "a2"])
    assert segs == [Segment(0, 0, 128, 3), Segment(2, 128, 192, 3), Segment(2, 192, 384, 4)]


def test_split_segments_respects_launch_limits():
    from paper_2510_00206_b200.plan import split_segments

    ads = [AdapterConfig(64) for _ in range(5)]
    segs = segments_from_lengths([0, 1, 2, 3, 4], [100, 50, 70, 30, 60], start=10)  # rows 10..320, m = 400
    parts = split_segments(ads, segs, 400)
    assert [(a, b) for a, b, _ in parts] == [(0, 160), (160, 260), (260, 400)]
    assert [[s.adapter for s in g] for _, _, g in parts] == [[0, 1], [2, 3], [4]]
    # segments of an adapter already in the group add no columns
    ads2 = [AdapterConfig(64), AdapterConfig(64), AdapterConfig(16)]
    segs2 = segments_from_lengths([0, 1, 0, 1, 2], [10, 10, 10, 10, 10])
    assert len(split_segments(ads2, segs2, 50)) == 2
    assert [len(g) for _, _, g in split_segments(ads2, segs2, 50)] == [4, 1]
    # everything fits: one range covering all rows
    assert split_segments([AdapterConfig(16)], [Segment(0, 5, 9)], 20) == [(0, 20, [Segment(0, 5, 9)])]
    # the segment-count limit
    many = [Segment(0, i, i + 1) for i in range(40)]
    assert [len(g) for _, _, g in split_segments([AdapterConfig(8)], many, 40)] == [32, 8]
    with pytest.raises(ValidationError):
        split_segments([AdapterConfig(200)], [Segment(0, 0, 4)], 4)


def test_module_dropout_state_round_trip_and_strict_state_dict():
    """Checkpoints: the Philox step is saved/restored explicitly (resumed runs continue the
    dropout stream), and the state dict holds only the PEFT-named tensors, so it loads
    strictly (CPU: no kernel runs)."""
    from paper_2510_00206_b200 import FusedLoRA, FusedMultiLoRA

    w = torch.zeros(64, 32, dtype=torch.bfloat16)
    a = FusedLoRA(w, rank=8, dropout_p=0.1, seed=3, dropout_rng="counter")
    a._offset = 17
    b = FusedLoRA(w.clone(), rank=8, dropout_p=0.1, seed=3, dropout_rng="counter")
    b.load_state_dict(a.state_dict(), strict=True)
    assert set(a.state_dict()) == {"lora_A.weight", "lora_B.weight"}
    b.load_dropout_state(a.dropout_state())
    assert b._offset == 17 and b.next_offset() == 17
    m = FusedMultiLoRA(w, [AdapterConfig(8), AdapterConfig(16)], dropout_rng="counter")
    m._offset = 5
    m2 = FusedMultiLoRA(w.clone(), [AdapterConfig(8), AdapterConfig(16)], dropout_rng="counter")
    m2.load_state_dict(m.state_dict(), strict=True)
    m2.load_dropout_state(m.dropout_state())
    assert m2._offset == 5 and torch.equal(m2.lora_B[1].weight, m.lora_B[1].weight)
    # torch-RNG offsets (the default) follow torch's RNG state instead: nothing to restore
    t = FusedLoRA(w.clone(), rank=8, dropout_p=0.1)
    assert t.dropout_rng == "torch" and t.dropout_state() == {"dropout_rng": "torch"}
    t.load_dropout_state({"philox_step": 3})
    with pytest.raises(ValidationError):
        FusedLoRA(w.clone(), rank=8, dropout_rng="numpy")


def test_frozen_base_bias_does_not_train():
    from paper_2510_00206_b200 import FusedLoRA

    base = torch.nn.Linear(32, 64, bias=True)
    layer = FusedLoRA(base, rank=8)
    assert not base.weight.requires_grad and not base.bias.requires_grad
    assert {n for n, p in layer.named_parameters() if p.requires_grad} == {"lora_A.weight", "lora_B.weight"}


def test_split_segments_counts_unshared_blocks_per_segment():
    """FusedMultiLoRA(track_slot_grads=True) gives every segment its own column block: the
    split must count a rank-64 adapter's three global batches as 192 columns."""
    segs = [Segment(0, 0, 100, 0), Segment(0, 100, 200, 1), Segment(0, 200, 300, 2)]
    assert len(split_segments([AdapterConfig(64)], segs, 300)) == 1
    parts = split_segments([AdapterConfig(64)], segs, 300, share_blocks=False)
    assert [(r0, r1, len(g)) for r0, r1, g in parts] == [(0, 200, 2), (200, 300, 1)]
    for r0, r1, g in parts:
        local = [Segment(s.adapter, s.row_start - r0, s.row_end - r0, s.batch) for s in g]
        LayerPlan(r1 - r0, 64, 64, [AdapterConfig(64)], local, share_blocks=False)  # fits one launch


def test_whole_microbatch_validation_has_no_segment_cap():
    """More than 32 segments are valid for a microbatch (fused_multi_lora splits it into
    launches); one launch's plan still enforces the cap."""
    segs = segments_from_lengths([0] * 40, [1] * 40)
    validate_segments(segs, 40, 1, max_segments=None)
    with pytest.raises(ValidationError):
        validate_segments(segs, 40, 1)


def test_group_module_names_and_validation():
    from paper_2510_00206_b200 import FusedLoRAGroup

    w = lambda n, k: torch.zeros(n, k, dtype=torch.bfloat16)  # noqa: E731
    g = FusedLoRAGroup({"q_proj": w(64, 32), "k_proj": w(16, 32), "v_proj": w(16, 32)}, rank=[16, 8, 8])
    assert [n for n, _ in g.named_parameters()] == [f"{p}.lora_{ab}.weight" for p in ("q_proj", "k_proj", "v_proj")
                                                    for ab in ("A", "B")]
    assert g.k_proj.config.rank == 8 and g.q_proj.config.seed == 0 and g.v_proj.config.seed == 2
    with pytest.raises(ValidationError):
        FusedLoRAGroup({"a": w(64, 32), "b": w(64, 16)}, rank=8)  # different inputs
    with pytest.raises(ValidationError):
        FusedLoRAGroup({"a": w(64, 32)}, rank=[8, 16])
