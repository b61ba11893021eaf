"""Schedule ingestion: lorasched schedule documents -> FusedMultiLoRA segment tables.

The reference's scheduler emits a versioned JSON document "consumed by the simulator and
by external training systems" (ls/schedule.py:441-490; reference SPEC.md:386). Each
``microbatch`` entry lists padded per-(adapter, global batch) segments in the order the
rows are packed (ls/packing.py:251-258). This module turns such a document (or
lorasched ``Microbatch`` objects directly) into :class:`~.plan.Segment` lists and
:class:`~.plan.AdapterConfig` tables for :class:`~.modules.FusedMultiLoRA` — SURVEY.md
§8(f) "next" #1. Validation mirrors ``schedule_from_doc`` (ls/schedule.py:499-550).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Any, Mapping, Sequence

from .errors import ValidationError
from .plan import AdapterConfig, Segment

SCHEDULE_SCHEMA_VERSION = 1  # ls/schedule.py:21
KIND_MICROBATCH = "microbatch"
KIND_NOOP = "noop"


def _padded(raw: int, multiple: int) -> int:
    return -(-int(raw) // int(multiple)) * int(multiple)


def _need(d: Mapping, key: str, where: str):
    if key not in d:
        raise ValidationError(f"{where}: missing field {key!r}")
    return d[key]


@dataclass(frozen=True)
class MicrobatchPlan:
    """One microbatch ready for the fused layer: its segments and total padded rows.

    ``sequences`` lists the row count of every packed sequence in row order: each sample
    of a segment, then (when the segment was padded) one pad pseudo-sequence of
    ``padded − raw`` rows, so varlen attention never mixes samples or attends into padding.
    ``segment_raw`` holds each segment's raw (unpadded) token count.
    """

    commit_index: int
    group_id: int
    segments: tuple
    rows: int
    raw_tokens: int
    sequences: tuple = ()
    segment_raw: tuple = ()


def adapters_from_doc(doc: Mapping, seeds: Mapping[str, int] | None = None) -> tuple[list[str], list[AdapterConfig]]:
    """Adapter ids (slot order) and configs from the document's ``adapters`` list."""
    ads = _need(doc, "adapters", "schedule")
    ids, cfgs = [], []
    for i, a in enumerate(ads):
        where = f"adapters[{i}]"
        aid = _need(a, "adapter_id", where)
        if aid in ids:
            raise ValidationError(f"{where}: duplicate adapter id {aid!r}")
        rank = int(_need(a, "lora_rank", where))
        alpha = float(_need(a, "alpha", where))
        p = float(a.get("dropout_p", 0.0))
        ids.append(aid)
        cfgs.append(AdapterConfig(rank=rank, scaling=alpha / rank, dropout_p=p,
                                  seed=int((seeds or {}).get(aid, 1000 + i))))
    return ids, cfgs


def microbatches_from_doc(doc: Mapping, adapter_ids: Sequence[str] | None = None) -> list[MicrobatchPlan]:
    """Every ``microbatch`` entry as a MicrobatchPlan (no-ops are skipped)."""
    ver = _need(doc, "schema_version", "schedule")
    if ver != SCHEDULE_SCHEMA_VERSION:
        raise ValidationError(f"schedule: unsupported schema_version {ver!r} (expected {SCHEDULE_SCHEMA_VERSION})")
    if adapter_ids is None:
        adapter_ids, _ = adapters_from_doc(doc)
    slot = {a: i for i, a in enumerate(adapter_ids)}
    out = []
    for i, e in enumerate(_need(doc, "entries", "schedule")):
        where = f"entries[{i}]"
        kind = _need(e, "kind", where)
        if kind == KIND_NOOP:
            continue
        if kind != KIND_MICROBATCH:
            raise ValidationError(f"{where}: unknown kind {kind!r}")
        row, raw_total, segs, seqs, seg_raw = 0, 0, [], [], []
        for j, s in enumerate(_need(e, "segments", where)):
            sw = f"{where}.segments[{j}]"
            aid = _need(s, "adapter_id", sw)
            if aid not in slot:
                raise ValidationError(f"{sw}: unknown adapter {aid!r}")
            mult = int(_need(s, "padding_multiple", sw))
            samples = _need(s, "samples", sw)
            lens = [int(_need(r, "length", f"{sw}.samples")) for r in samples]
            if any(n < 1 for n in lens):
                raise ValidationError(f"{sw}.samples: lengths must be >= 1")
            raw = sum(lens)
            padded = _padded(raw, mult)
            seqs.extend(lens)
            seg_raw.append(raw)
            if padded > raw:
                seqs.append(padded - raw)
            declared = s.get("padded_tokens")
            if declared is not None and int(declared) != padded:
                raise ValidationError(f"{sw}.padded_tokens: declared {declared}, recomputed {padded}")
            segs.append(Segment(slot[aid], row, row + padded, int(_need(s, "global_batch_index", sw))))
            row += padded
            raw_total += raw
        declared = e.get("total_padded_tokens")
        if declared is not None and int(declared) != row:
            raise ValidationError(f"{where}.total_padded_tokens: declared {declared}, recomputed {row}")
        out.append(MicrobatchPlan(int(e.get("commit_index", i)), int(_need(e, "group_id", where)), tuple(segs), row,
                                  raw_total, tuple(seqs), tuple(seg_raw)))
    return out


def segments_from_microbatch(mb: Any, adapter_ids: Sequence[str]) -> list[Segment]:
    """Segments of a lorasched ``Microbatch`` object (ls/packing.py:63-98), duck-typed."""
    slot = {a: i for i, a in enumerate(adapter_ids)}
    row, segs = 0, []
    for s in mb.segments:
        if s.adapter_id not in slot:
            raise ValidationError(f"unknown adapter {s.adapter_id!r}")
        n = int(s.padded_tokens)
        segs.append(Segment(slot[s.adapter_id], row, row + n, int(s.global_batch_index)))
        row += n
    return segs
