"""The traffic-model mirror equals the reference's own numbers (pinned by fixtures
generated from lorasched itself, tests/golden/make_reference_golden.py)."""
from __future__ import annotations

import json
import os
import warnings

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import traffic as otraffic
from paper_2510_00206_b200 import costmodel as T

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "traffic_reference.json")))


def _shape(m, k, n, r, e):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return T.GemmShape(m=m, k=k, n=n, r=r, element_bytes=e)


@pytest.mark.parametrize("row", GOLD["reports"], ids=lambda r: f"{r['shape']}-{r['variant']}-{r['pass']}")
def test_report_matches_reference(row):
    m, k, n, r, e = row["shape"]
    rep = T.traffic(_shape(m, k, n, r, e), row["pass"], row["variant"])
    assert rep.to_dict() == row["report"]
    # the oracle's independent count agrees kernel by kernel
    ok = otraffic.kernels(m, k, n, r, e, row["variant"], row["pass"])
    assert [(kk["kernel"], kk["bytes_read"], kk["bytes_written"]) for kk in row["report"]["kernels"]] == ok


def test_frozen_reference_totals():
    ft = GOLD["frozen_totals"]  # pkg/tests/test_costmodel.py:22-27
    s = T.GemmShape(8192, 4096, 4096, 16)
    assert T.roundtrip_bytes(s, "unfused") == ft["REF_UNFUSED_TOTAL"]
    assert T.roundtrip_bytes(s, "fused_lora") == ft["REF_FUSED_TOTAL"]
    assert T.roundtrip_bytes(T.GemmShape(8192, 4096, 4096, 0), "unfused") == ft["REF_FROZEN_TOTAL"]
    assert 2.4 <= ft["REF_UNFUSED_TOTAL"] / ft["REF_FROZEN_TOTAL"] <= 2.9
    assert 0.60 <= ft["REF_FUSED_TOTAL"] / ft["REF_UNFUSED_TOTAL"] <= 0.68


def test_service_response_fields_reproduce():
    body = GOLD["service_traffic_unfused"]  # POST /v1/traffic, pkg/tests/test_service.py:140-150
    s = T.GemmShape(8192, 4096, 4096, 16)
    assert body["total_bytes"] == T.roundtrip_bytes(s, "unfused")
    assert body["baseline_total_bytes"] == T.roundtrip_bytes(T.GemmShape(8192, 4096, 4096, 0), "unfused")
    assert body["arithmetic_intensity"] == pytest.approx(T.arithmetic_intensity(16, 4096, 8192))
    assert body["memory"] == T.lora_memory_bytes(4096, 4096, 16).to_dict()
    assert body["forward"] == T.traffic(s, "forward", "unfused").to_dict()
    multi = GOLD["service_traffic_multi"]
    assert multi["backward"] == T.traffic(s, "backward", "fused_multi_lora").to_dict()


def test_eq2_and_memory():
    assert T.arithmetic_intensity(16, 4096, 8192) == pytest.approx(GOLD["eq2_reference"])
    assert T.arithmetic_intensity(16, 4096, 8192) == pytest.approx(15.907, abs=1e-3)
    assert T.lora_memory_bytes(4096, 4096, 16).to_dict() == GOLD["memory_reference"]
    assert T.H100_SXM.machine_balance == pytest.approx(295.2, abs=0.5)
    assert T.B200.machine_balance == pytest.approx(1611.4e12 / 6532.9e9)


def test_b200_minimal_formulas():
    """K1 = 2mk+2kr+2mr, K2 = 2(mk+kn+mr+rn)+2mn, K3 = 2(mn+rn+mr)+2mr+4rn,
    K4 = 2(mk+mr)+4kr, K5 = 2(mn+kn+mr+kr)+2mk."""
    m, k, n, r = 2048, 4096, 4096, 16
    s = T.GemmShape(m, k, n, r)
    fwd = {kk.kernel: kk.total_bytes for kk in T.traffic(s, "forward", "b200_minimal").kernels}
    bwd = {kk.kernel: kk.total_bytes for kk in T.traffic(s, "backward", "b200_minimal").kernels}
    assert fwd["dropout_down_proj_fused"] == 2 * m * k + 2 * k * r + 2 * m * r
    assert fwd["base_gemm_epilogue_fused"] == 2 * (m * k + k * n + m * r + r * n) + 2 * m * n
    assert bwd["grad_up_fused"] == 2 * (m * n + r * n + m * r) + 2 * m * r + 4 * r * n
    assert bwd["grad_down_fused"] == 2 * (m * k + m * r) + 4 * k * r
    assert bwd["grad_base_accum_fused"] == 2 * (m * n + k * n + m * r + k * r) + 2 * m * k
    # SURVEY.md §8(d) C1 total: 186.0 MB
    total = T.roundtrip_bytes(s, "b200_minimal")
    assert abs(total / 1e6 - 186.0) < 0.5


def test_b200_built_adds_the_packed_keep_mask():
    """b200_built = b200_minimal + the bit-packed keep mask: written by ①, read by ④ and ⑤."""
    m, k, n, r = 2048, 4100, 4096, 16
    s = T.GemmShape(m, k, n, r)
    bits = m * ((k + 7) // 8)
    for ps in ("forward", "backward"):
        mini = {kk.kernel: (kk.bytes_read, kk.bytes_written) for kk in T.traffic(s, ps, "b200_minimal").kernels}
        built = {kk.kernel: (kk.bytes_read, kk.bytes_written) for kk in T.traffic(s, ps, "b200_built").kernels}
        assert mini.keys() == built.keys()
        for name, (rd, wr) in built.items():
            drd, dwr = rd - mini[name][0], wr - mini[name][1]
            want = {"dropout_down_proj_fused": (0, bits), "grad_down_fused": (bits, 0),
                    "grad_base_accum_fused": (bits, 0)}.get(name, (0, 0))
            assert (drd, dwr) == want, name
    assert T.roundtrip_bytes(s, "b200_built") - T.roundtrip_bytes(s, "b200_minimal") == 3 * bits
    for ps in ("forward", "backward"):  # the oracle's independent restatement agrees
        ours = [(kk.kernel, kk.bytes_read, kk.bytes_written) for kk in T.traffic(s, ps, "b200_built").kernels]
        assert ours == [tuple(x) for x in otraffic.kernels(m, k, n, r, 2, "b200_built", ps)]


@given(m=st.integers(1, 1 << 14), k=st.integers(1, 1 << 13), n=st.integers(1, 1 << 13), r=st.integers(1, 64))
@settings(max_examples=100, deadline=None)
def test_b200_design_never_exceeds_reference_fused(m, k, n, r):
    """The built design differs from the reference's fused model by rank-sized terms only:
    ours − ref = 2r(m+k+n) − 8mk (it drops the stored mask, X̂ and the mk-sized LoRA
    input-gradient), so it moves strictly less whenever r(m+k+n) < 4mk."""
    s = _shape(m, k, n, r, 2)
    ours, ref = T.roundtrip_bytes(s, "b200_minimal"), T.roundtrip_bytes(s, "fused_lora")
    assert ours - ref == 2 * r * (m + k + n) - 8 * m * k
    if r * (m + k + n) < 4 * m * k:
        assert ours < ref


def test_validation_errors():
    with pytest.raises(ValueError):
        T.traffic(T.GemmShape(8, 8, 8, 1), "sideways", "unfused")
    with pytest.raises(ValueError):
        T.traffic(T.GemmShape(8, 8, 8, 1), "forward", "bogus")
    with pytest.raises(ValueError):
        T.GemmShape(0, 8, 8, 1)
    with pytest.raises(ValueError):
        T.HardwareProfile(1e15, 4e12, machine_balance=100.0)
    with pytest.warns(UserWarning, match="rank"):
        T.GemmShape(m=16, k=8, n=8, r=32)


def test_flops_formula():
    f = T.lora_flops(2048, 4096, 4096, 16)
    assert f["total"] == 4 * 2048 * 4096 * 4096 + 6 * 2048 * 16 * (4096 + 4096)
    assert abs(f["total"] - 1.3905e11) / 1.3905e11 < 1e-3
