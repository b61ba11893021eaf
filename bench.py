"""Benchmark of the FusedLoRA hot path (BASELINE.json metric) — one JSON line on rank 0.

Metric: "LoRA linear fwd+bwd tokens/s & TFLOP/s (8B/70B shapes), % of bf16 peak".
Workload (default, BASELINE.json configs[1]): one step = forward + backward of the seven
LLaMa-3.1-8B LoRA linears (q, k, v, o, gate, up, down; hidden 4096, kv 1024, ffn 14336),
r = 16, scaling 2.0, dropout p = 0.1, 8192 tokens per GPU, bf16, frozen W, random init,
synthetic inputs. q/k/v share the attention input and gate/up the MLP input, as in the
decoder. With N GPUs (torchrun, one process per GPU) every rank runs its own 8192 tokens
(weak scaling, data parallel) and the fp32 dA/dB of all seven adapters are NCCL
all-reduced once per step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c1|c4] [--impl ours|reference]

`--impl reference` times the reference CPU path of this hot path (the oracle port in
oracle/, numpy, all host threads) on a bounded token sample of the same workload.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HIDDEN_8B, KV_8B, FFN_8B = 4096, 1024, 14336
HIDDEN_70B, KV_70B, FFN_70B = 8192, 1024, 28672


def projections(config: str):
    """(name, k, n, input group) of each LoRA linear of one decoder layer."""
    if config in ("c2", "c1", "c3", "c5"):
        h, kv, f = HIDDEN_8B, KV_8B, FFN_8B
    elif config == "c4":
        h, kv, f = HIDDEN_70B, KV_70B, FFN_70B
    else:
        raise SystemExit(f"unknown config {config}")
    if config == "c1":
        return [("linear", 4096, 4096, "x")]
    return [("q", h, h, "attn"), ("k", h, kv, "attn"), ("v", h, kv, "attn"), ("o", h, h, "o"),
            ("gate", h, f, "mlp"), ("up", h, f, "mlp"), ("down", f, h, "down")]


TOKENS_OVERRIDE: int | None = None  # --tokens


def tokens_per_gpu(config: str, world: int = 1) -> int:
    """Tokens each rank processes per step. C4 is strong-scaled (BASELINE configs[3], SURVEY
    §8(d)): 16384 tokens per step in total, 16384 / N per rank; the others are weak-scaled
    (a fixed per-GPU batch)."""
    if TOKENS_OVERRIDE:
        return TOKENS_OVERRIDE
    if config == "c4":
        if 16384 % world:
            raise SystemExit(f"--config c4 strong-scales 16384 tokens: N={world} must divide it")
        return 16384 // world
    return {"c1": 2048, "c2": 8192, "c3": 8192, "c5": 8192}[config]


def scaling_kind(config: str) -> str:
    return "strong" if config == "c4" and not TOKENS_OVERRIDE else "weak"


# C3 (BASELINE.json configs[2]): FusedMultiLoRA, 4 adapters of ranks
# 8/16/32/64 (scaling 2.0, p = 0/0.05/0.1/0.1, seeds 1..4) on uneven tile-aligned segments
C3_RANKS = (8, 16, 32, 64)
C3_DROPOUT = (0.0, 0.05, 0.1, 0.1)
C3_LENGTHS = (3584, 2432, 1408, 768)


def c3_adapters():
    from paper_2510_00206_b200 import AdapterConfig

    return [AdapterConfig(rank=r, scaling=2.0, dropout_p=p, seed=i + 1)
            for i, (r, p) in enumerate(zip(C3_RANKS, C3_DROPOUT))]


def c3_segments():
    from paper_2510_00206_b200 import segments_from_lengths

    return segments_from_lengths(range(len(C3_LENGTHS)), C3_LENGTHS)


def c3_flops(m: int) -> float:
    """4mkn + 6 Σ_seg rows·r·(k+n) over the 7 projections."""
    return float(sum(4 * m * k * n + sum(6 * L * r * (k + n) for L, r in zip(C3_LENGTHS, C3_RANKS))
                     for _, k, n, _ in projections("c3")))


def step_flops(config: str, m: int, r: int) -> float:
    if config == "c3":
        return c3_flops(m)
    return float(sum(4 * m * k * n + 6 * m * r * (k + n) for _, k, n, _ in projections(config)))


def gemm_flops(config: str, m: int, r: int) -> dict:
    """Algorithmic FLOPs of the two tcgen05 GEMM launchers per step."""
    if config == "c3":
        lr = sum(L * rr for L, rr in zip(C3_LENGTHS, C3_RANKS))
        fwd = sum(2 * m * k * n + 2 * lr * n for _, k, n, _ in projections(config))
        dgrad = sum(2 * m * n * k + 2 * lr * k for _, k, n, _ in projections(config))
        return {"base_fwd": float(fwd), "grad_input": float(dgrad)}
    fwd = sum(2 * m * k * n + 2 * m * r * n for _, k, n, _ in projections(config))
    dgrad = sum(2 * m * n * k + 2 * m * r * k for _, k, n, _ in projections(config))
    return {"base_fwd": float(fwd), "grad_input": float(dgrad)}


def lowrank_bytes(config: str, m: int, r: int) -> dict:
    """Algorithmic HBM bytes of the memory-bound launchers per step;
    C3: r = the padded rank-concat width the kernels stream (Σ padded ranks = 128)."""
    if config == "c3":
        r = 128
    k1 = sum(2 * m * k + 2 * k * r + 2 * m * r for _, k, n, _ in projections(config))
    k3 = sum(2 * (m * n + r * n + m * r) + 2 * m * r + 4 * r * n for _, k, n, _ in projections(config))
    k4 = sum(2 * (m * k + m * r) + 4 * k * r for _, k, n, _ in projections(config))
    return {"dropout_down_fwd": float(k1), "grad_up": float(k3), "grad_down": float(k4)}


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                "bf16_tflops_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                "source": "MEASURED_PEAKS.json (measured)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "source": "B200_PROFILING.md fallback"}


def gemm_traffic(config: str = "c2") -> dict | None:
    """DRAM bytes per lf_gemm_kernel launch from the committed ncu capture of one bench step
    of this config (tools/ncu_traffic.py -> profiles/gemm_traffic.json for C2,
    profiles/gemm_traffic_<config>.json otherwise), or None when there is none."""
    name = "gemm_traffic.json" if config == "c2" else f"gemm_traffic_{config}.json"
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return json.load(f)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------------------
# reference arm: the CPU oracle (numpy port) on the host cores
# --------------------------------------------------------------------------------------
_CPU_INPUTS: dict = {}


def _cpu_inputs(config: str, sample_tokens: int, r: int):
    """Seeded bf16-valued inputs of every projection for the CPU leg (generated once: the
    weight matrices take longer to draw than the sample takes to compute)."""
    import numpy as np

    from oracle import lora as olora

    key = (config, sample_tokens, r)
    if key not in _CPU_INPUTS:
        rng = np.random.default_rng(0)
        xs, out = {}, []
        for name, k, n, grp in projections(config):
            m = sample_tokens
            if grp not in xs:
                xs[grp] = olora.bf16_round(rng.standard_normal((m, k), dtype=np.float32))
            w = olora.bf16_round(rng.standard_normal((n, k), dtype=np.float32) / np.sqrt(k))
            a = olora.bf16_round((rng.random((r, k), dtype=np.float32) * 2 - 1) / np.sqrt(k))
            b = olora.bf16_round(rng.standard_normal((n, r), dtype=np.float32) / np.sqrt(r))
            dy = olora.bf16_round(rng.standard_normal((m, n), dtype=np.float32))
            out.append((k, xs[grp], w, a, b, dy))
        _CPU_INPUTS[key] = out
    return _CPU_INPUTS[key]


def cpu_reference_step(config: str, sample_tokens: int, r: int, p: float, step: int = 0,
                       acc: str = "float32") -> float:
    """One fwd+bwd of every projection on a `sample_tokens`-row sample with the oracle's
    algorithm (oracle/lora.py: Philox keep mask, Eq. 1 at SPEC §2's rounding points) at
    `acc` accumulation; returns the wall seconds of the compute (input generation excluded).
    Each step draws its own dropout mask (Philox offset = step)."""
    import numpy as np

    from oracle import lora as olora
    from oracle import philox as ophilox

    dt = np.float32 if acc == "float32" else np.float64
    total = 0.0
    for k, x, w, a, b, dy in _cpu_inputs(config, sample_tokens, r):
        m = x.shape[0]
        seg = [olora.OracleSegment(0, m, 0, r, 2.0, p, 1234)]
        t1 = time.perf_counter()
        keep = ophilox.keep_mask_rows(np.arange(m), k, p, 1234, step)
        y, s_hat = olora.forward(x, w, a, b, seg, keep, acc=dt)
        olora.backward(dy, x, w, a, b, s_hat, seg, keep, acc=dt)
        total += time.perf_counter() - t1
    return total


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def cpu_torch_c1(repeats: int = 3) -> dict:
    """SURVEY §8(d) baseline 3: the unfused LoRA linear (baseline.unfused_lora) in fp32 torch
    on the host cores at C1 (2048 tokens, k = n = 4096, r = 16, p = 0.1, W frozen), forward +
    backward with autograd, best of `repeats` after one warm-up."""
    import torch

    from paper_2510_00206_b200.baseline import unfused_lora

    g = torch.Generator().manual_seed(0)
    m, k, n, r = 2048, 4096, 4096, 16
    x = torch.randn(m, k, generator=g).requires_grad_(True)
    w = torch.randn(n, k, generator=g) / k**0.5
    a = ((torch.rand(r, k, generator=g) * 2 - 1) / k**0.5).requires_grad_(True)
    b = (torch.randn(n, r, generator=g) / r**0.5).requires_grad_(True)
    dy = torch.randn(m, n, generator=g)
    best = float("inf")
    for i in range(repeats + 1):
        t0 = time.perf_counter()
        unfused_lora(x, w, a, b, 2.0, 0.1, training=True).backward(dy)
        dt_ = time.perf_counter() - t0
        x.grad = a.grad = b.grad = None
        if i:
            best = min(best, dt_)
    flops = 4 * m * k * n + 6 * m * r * (k + n)
    return {"ms_per_step": best * 1e3, "tokens_per_s": m / best, "tflops": flops / best / 1e12,
            "threads": torch.get_num_threads(), "cpu": cpu_model(),
            "what": "fp32 torch-CPU unfused LoRA linear (F.linear + F.dropout + add/scale, autograd, W frozen), "
                    "C1: 2048 tokens, k=n=4096, r=16, p=0.1; best of 3 after warm-up"}


def run_reference(args, rank: int, world: int) -> None:
    """--impl reference: the reference CPU path of this hot path — the oracle port
    (oracle/lora.py, the algorithm the reference's kernel list specifies) — on the host
    cores, on a bounded token sample of this arm's workload; same metric, unit and config."""
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    sample = args.cpu_sample_tokens
    r, p = 16, args.dropout
    # torchrun sets OMP_NUM_THREADS=1 for N > 1: rank 0 alone runs the reference here, on every
    # host thread it may use
    from threadpoolctl import threadpool_limits

    with threadpool_limits(limits=cores):
        for _ in range(max(1, min(args.warmup, 1))):
            cpu_reference_step(args.config, 64, r, p)
        times = [cpu_reference_step(args.config, sample, r, p, step=i) for i in range(args.steps)]
    t = sum(times) / len(times)
    value = sample / t
    line = {
        "impl": "reference",
        "metric": "LoRA linear fwd+bwd tokens/s & TFLOP/s (8B/70B shapes), % of bf16 peak",
        "value": value,
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t * 1e3,
        "higher_is_better": True,
        "scaling": scaling_kind(args.config),
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic",
        "config": bench_config(args.config, world, r, p),
        "execution": f"CPU, {cores} host threads (numpy BLAS), rank 0 only",
        "tflops": step_flops(args.config, sample, r) / t / 1e12,
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "port", "cpu": cpu_model(),
                         "sample": f"{sample} tokens of each projection per step, fwd+bwd, oracle/lora.py at fp32 "
                                   "accumulation with its Philox keep mask (oracle/philox.py)"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def bench_config(config: str, world: int, r: int, p: float) -> dict:
    """The `config` object both arms print (the driver compares them)."""
    m = tokens_per_gpu(config, world)
    return {
        "workload": workload_name(config, world),
        "projections": [[nm, k, n] for nm, k, n, _ in projections(config)],
        "tokens_per_gpu": m,
        "global_tokens": m * world,
        "rank": list(C3_RANKS) if config == "c3" else r,
        "scaling": 2.0,
        "dropout_p": list(C3_DROPOUT) if config == "c3" else p,
        "parallelism": f"dp{world}",
        "l2": "inputs larger than L2 (≈2 GB touched per step vs 126 MB L2)",
    }


def workload_name(config: str, world: int = 1) -> str:
    m = tokens_per_gpu(config, world)
    gpus = f"{world} B200" + ("" if world == 1 else " data-parallel")
    return {
        "c2": f"LLaMa-3.1-8B layer shapes (q/k/v/o, gate/up/down) FusedLoRA r=16, {m} tokens per GPU, bf16, {gpus}",
        "c1": f"single FusedLoRA linear fwd+bwd: tokens={m} per GPU, k=n=4096, r=16, dropout=0.1, {gpus}",
        "c4": (f"LLaMa-3.1-70B layer shapes (k=8192, n=28672) FusedLoRA r=16, {m * world} tokens per step "
               f"({m} per GPU, {scaling_kind(config)} scaling), bf16, {gpus}"),
        "c5": f"LLaMa-3.1-8B 4 concurrent LoRA jobs, full decoder fwd+bwd step, {gpus}",
        "c3": f"FusedMultiLoRA 4 adapters, ranks {{8,16,32,64}}, uneven token segments {{3584,2432,1408,768}} "
              f"sharing one frozen W per projection (LLaMa-3.1-8B q/k/v/o/gate/up/down), {m} tokens per GPU, {gpus}",
    }[config]


# --------------------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------------------
def build_layers(config: str, m: int, r: int, p: float, device, gen, capturable: bool = False):
    import torch

    from paper_2510_00206_b200 import FusedLoRA, FusedMultiLoRA

    layers, inputs, grads = {}, {}, {}
    for i, (name, k, n, grp) in enumerate(projections(config)):
        w = (torch.randn(n, k, generator=gen, device=device, dtype=torch.float32) / k**0.5).to(torch.bfloat16)
        if config == "c3":
            adapters = [dataclasses.replace(a, seed=a.seed + 100 * i) for a in c3_adapters()]
            layer = FusedMultiLoRA(w, adapters, init="gaussian", generator=gen, capturable=capturable).to(device)
        else:
            layer = FusedLoRA(w, rank=r, scaling=2.0, dropout_p=p, seed=1234 + i, init="gaussian",
                              generator=gen, capturable=capturable).to(device)
        layers[name] = layer
        if grp not in inputs:
            # activations come from the previous layer: they need dX (⑤ runs every step)
            inputs[grp] = torch.randn(m, k, generator=gen, device=device, dtype=torch.float32).to(
                torch.bfloat16).requires_grad_(True)
        grads[name] = torch.randn(m, n, generator=gen, device=device, dtype=torch.float32).to(torch.bfloat16)
    return layers, inputs, grads


def layer_call(config: str):
    """How a step calls one layer: FusedLoRA(x), or FusedMultiLoRA(x, segments) for C3."""
    if config == "c3":
        segs = c3_segments()
        return lambda layer, x: layer(x, segs)
    return lambda layer, x: layer(x)


def adapter_params(layers):
    return [p for nm in layers for p in layers[nm].parameters() if p.requires_grad]


# projections that read the same input in a decoder layer: run as one FusedLoRAGroup
# (SURVEY §8(f)#4 — the input gradient is summed inside the ⑤ GEMM epilogues)
SHARED_INPUT_GROUPS = ("attn", "mlp")
GROUPED = True  # --no-group: every projection as its own FusedLoRA call
_UNITS: dict = {}


def step_units(config: str, layers: dict):
    """How one step calls the layers: [(group input, [names], module or FusedLoRAGroup)]."""
    from paper_2510_00206_b200 import FusedLoRAGroup, FusedMultiLoRAGroup

    cache = _UNITS
    key = (id(layers), config, GROUPED)
    if key not in cache:
        units, by_grp = [], {}
        for name, k, n, grp in projections(config):
            by_grp.setdefault(grp, []).append(name)
        for grp, names in by_grp.items():
            if GROUPED and grp in SHARED_INPUT_GROUPS and len(names) > 1:
                kind = FusedMultiLoRAGroup if config == "c3" else FusedLoRAGroup
                units.append((grp, names, kind.from_layers({nm: layers[nm] for nm in names})))
            else:
                units.extend((grp, [nm], layers[nm]) for nm in names)
        cache[key] = units
    return cache[key]


def fused_step(config, layers, inputs, grads, world, flat_grad=None):
    """fwd+bwd of every projection through the public module API; grads all-reduced if world>1."""
    import torch

    call = layer_call(config)
    for grp, names, mod in step_units(config, layers):
        if len(names) > 1:
            ys = call(mod, inputs[grp])
            torch.autograd.backward(ys, [grads[nm] for nm in names])
        else:
            y = call(mod, inputs[grp])
            y.backward(grads[names[0]])
    if world > 1:
        allreduce_grads(layers)


def allreduce_grads(layers):
    """The one data-parallel exchange: SUM all-reduce of the flat fp32 adapter gradients."""
    import torch
    import torch.distributed as dist

    params = adapter_params(layers)
    flat = torch.cat([p.grad.reshape(-1) for p in params])
    dist.all_reduce(flat)
    off = 0
    for p in params:
        n_ = p.numel()
        p.grad.copy_(flat[off:off + n_].view_as(p))
        off += n_


def graphed_runner(step_local, world, layers, warmup):
    """One CUDA graph for the rank-local fwd+bwd; the NCCL all-reduce (world > 1) runs
    eagerly after each replay, so no collective is ever captured."""
    from paper_2510_00206_b200.graphs import GraphedStep

    g = GraphedStep(step_local, warmup=warmup)
    if world == 1:
        def run():
            return g.replay()
    else:
        def run():
            g.replay()
            allreduce_grads(layers)

    run.graphed = g  # the per-launcher timing pass captures beside it in the same memory pool
    return run


def graph_launch_durations(step_local, graphed, steps: int) -> dict:
    """{launcher: [ms per launch, ...]} over `steps` replays of a graph of the step captured
    with timing events around every launcher (external events: recorded inside the graph)."""
    import torch

    from paper_2510_00206_b200 import functional as F_
    from paper_2510_00206_b200.functional import refresh_stale_operand_shadows

    stats = F_.LaunchStats(timed=True, external=True)
    F_.set_launch_stats(stats)
    try:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, pool=graphed.graph.pool()):
            step_local()
    finally:
        F_.set_launch_stats(None)
    out: dict = {}
    for _ in range(steps):
        refresh_stale_operand_shadows()
        g.replay()
        torch.cuda.synchronize()
        for name, pairs in stats.events.items():
            out.setdefault(name, []).extend(a.elapsed_time(b) for a, b in pairs)
    del g
    return out


def zero_grads(layers, inputs=None):
    for p in adapter_params(layers):
        p.grad = None
    for t in (inputs or {}).values():
        t.grad = None


def unfused_base(config, layers):
    """bf16 copies of the adapter weights for the unfused torch arm: name -> (W, [A], [B])."""
    import torch

    base = {}
    for name, k, n, grp in projections(config):
        layer = layers[name]
        la = layer.lora_A if config == "c3" else [layer.lora_A]
        lb = layer.lora_B if config == "c3" else [layer.lora_B]
        a = [m_.weight.detach().to(torch.bfloat16).clone().requires_grad_(True) for m_ in la]
        b = [m_.weight.detach().to(torch.bfloat16).clone().requires_grad_(True) for m_ in lb]
        base[name] = (layer.base_weight, a, b)
    return base


def unfused_step(config, base, inputs, grads, p):
    """PEFT-style torch LoRA: cuBLAS F.linear + F.dropout + add/scale, autograd, W frozen
    (C3: the per-segment multi-adapter loop)."""
    from paper_2510_00206_b200 import unfused_lora, unfused_multi_lora

    for name, k, n, grp in projections(config):
        w, a, b = base[name]
        if config == "c3":
            y = unfused_multi_lora(inputs[grp], w, a, b, c3_adapters(), c3_segments(), training=True)
        else:
            y = unfused_lora(inputs[grp], w, a[0], b[0], 2.0, p, training=True)
        y.backward(grads[name])
        for t in a + b:
            t.grad = None


_KERNEL_CLASSES = (
    ("lf_gemm_kernel<false", "② base_fwd (lf_gemm_kernel, K-major W)"),
    ("lf_gemm_kernel<true", "⑤ grad_input (lf_gemm_kernel, MN-major W)"),
    ("lf_down_kernel", "① dropout_down_fwd (lf_down_kernel)"),
    ("lf_gradup_kernel", "③ grad_up (lf_gradup_kernel)"),
    ("lf_finalize_kernel", "③ grad_up dŜ finalize (lf_finalize_kernel)"),
    ("lf_dgrad_a_kernel", "④ grad_down (lf_dgrad_a_kernel)"),
    ("lf_routes_kernel", "routing table (lf_routes_kernel)"),
    ("distribution", "torch: dropout offset draw (randint)"),
    ("fill", "torch: zero-fill of the fp32 dA/dB accumulators"),
    ("elementwise", "torch: elementwise (fp32->bf16 operand casts, gradient sums, counters)"),
)


def step_breakdown(run, steps: int = 1) -> dict:
    """Where one step's device time goes: CUPTI kernel records of `steps` replays, each
    kernel credited with the time it extends the covered part of the timeline (programmatic
    dependent launch overlaps neighbours), gaps as `idle` — the parts sum to the span."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            run()
        torch.cuda.synchronize()
    evs = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
                  and not e.name.startswith(("Memcpy", "Memset"))), key=lambda e: e.time_range.start)
    if not evs:
        return {}
    parts: dict = {}
    t0 = evs[0].time_range.start
    covered = t0
    idle = 0.0
    for e in evs:
        a, b = e.time_range.start, e.time_range.end
        if a > covered:
            idle += a - covered
        gain = max(0.0, b - max(a, covered))
        covered = max(covered, b)
        name = next((lbl for key, lbl in _KERNEL_CLASSES if key in e.name), "other: " + e.name[:48])
        ent = parts.setdefault(name, [0, 0.0])
        ent[0] += 1
        ent[1] += gain
    span = covered - t0
    if os.environ.get("LF_BREAKDOWN_NAMES"):  # raw kernel names behind the classes (stderr)
        raw: dict = {}
        for e in evs:
            ent = raw.setdefault(e.name[:160], [0, 0.0])
            ent[0] += 1
            ent[1] += e.time_range.end - e.time_range.start
        for nm, (cnt, us) in sorted(raw.items(), key=lambda kv: -kv[1][1]):
            print(f"[breakdown] {us / steps:9.1f} us  x{cnt / steps:g}  {nm}", file=sys.stderr)
    out = {nm: {"ms_per_step": v[1] / 1e3 / steps, "kernels_per_step": v[0] / steps}
           for nm, v in sorted(parts.items(), key=lambda kv: -kv[1][1])}
    out["idle (gaps between kernels)"] = {"ms_per_step": idle / 1e3 / steps}
    return {"span_ms_per_step": span / 1e3 / steps, "parts": out,
            "method": "torch.profiler (CUPTI) over one graph replay after the timed loop; overlapping kernels "
                      "(PDL) credited with the time each extends the timeline, so parts + idle = span"}


def time_loop(fn, steps, warmup, sync_barrier):
    import torch

    for _ in range(warmup):
        fn()
    sync_barrier()
    torch.cuda.synchronize()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    for _ in range(steps):
        fn()
    stop.record()
    torch.cuda.synchronize()
    sync_barrier()
    return start.elapsed_time(stop) / steps


def run_ours(args, rank: int, world: int, local_rank: int) -> None:
    import torch
    import torch.distributed as dist

    from paper_2510_00206_b200 import _lib
    from paper_2510_00206_b200 import functional as F_

    _lib.load()  # fail loudly without the sm_100a library
    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    gen = torch.Generator(device=device).manual_seed(1000 + rank)
    r, p = 16, args.dropout
    m = tokens_per_gpu(args.config, world)
    layers, inputs, grads = build_layers(args.config, m, r, p, device, gen, capturable=args.graph)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], device=device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def step():
        zero_grads(layers, inputs)
        fused_step(args.config, layers, inputs, grads, world)

    def step_local():
        zero_grads(layers, inputs)
        fused_step(args.config, layers, inputs, grads, 1)

    # ---- device-resident timed region (value) ----------------------------------------
    # launch counting is host-side only (no events): one eager step, before any capture
    counts = F_.LaunchStats(timed=False)
    F_.set_launch_stats(counts)
    step()
    F_.set_launch_stats(None)
    launches = counts.total_launches() * args.steps
    if args.graph:
        # the whole fwd+bwd step (all projections, and the all-reduce when world > 1) as
        # one CUDA graph: the host leaves the loop (capturable layers: device Philox counter)
        try:
            run = graphed_runner(step_local, world, layers, args.warmup)
        except Exception as e:  # e.g. a collective that cannot be captured: time eagerly
            print(f"[bench] CUDA-graph capture failed ({type(e).__name__}: {e}); timing eagerly", file=sys.stderr)
            args.graph = False
            run = step
    else:
        run = step
    for _ in range(args.warmup):
        run()
    clocks = ClockSampler(local_rank)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(args.steps):
        run()
    t1.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    barrier()
    ms = max_over_ranks(t0.elapsed_time(t1) / args.steps)
    # per-launcher CUDA-event timing in a separate pass over the same steps (events on the
    # launching stream bracket every launcher; kept out of the headline loop). Graphed runs
    # capture the step once more with the events inside the graph, so each launcher is timed
    # on the device as it runs in the graph (an eager pass would add the host's launch gaps
    # to every small kernel: C1's GEMMs read 0.56 of peak that way)
    durs = None
    per_kernel_timing = "CUDA events around each launcher, eager steps"
    if args.graph and getattr(run, "graphed", None) is not None:
        try:
            durs = graph_launch_durations(step_local, run.graphed, args.steps)
            per_kernel_timing = "CUDA events around each launcher inside a CUDA-graph capture of the step"
        except Exception as e:
            print(f"[bench] graphed launcher timing failed ({type(e).__name__}: {e}); timing eagerly", file=sys.stderr)
    if durs is None:
        stats = F_.LaunchStats(timed=True)
        F_.set_launch_stats(stats)
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize()
        F_.set_launch_stats(None)
        durs = stats.durations_ms()

    breakdown = None
    if True:  # every rank replays (the replay may hold a collective)
        try:
            breakdown = step_breakdown(run)
        except Exception as e:  # profiler unavailable: the line still stands without it
            print(f"[bench] step breakdown failed ({type(e).__name__}: {e})", file=sys.stderr)

    # ---- per-kernel roofline ----------------------------------------------------------
    peaks = measured_peaks()
    gfl = gemm_flops(args.config, m, r)
    lrb = lowrank_bytes(args.config, m, r)
    kernels = {}
    for name, lst in durs.items():
        tot = sum(lst) / args.steps  # ms per step spent in this launcher
        ent = {"ms_per_step": tot, "launches_per_step": len(lst) / args.steps}
        if name in gfl:
            ent["tflops"] = gfl[name] / (tot * 1e-3) / 1e12
        if name in lrb:
            ent["gbs"] = lrb[name] / (tot * 1e-3) / 1e9
        kernels[name] = ent
    for name, ent in kernels.items():
        if name in lrb:
            ent["frac_of_hbm"] = ent["gbs"] / peaks["hbm_gbs"]
    if p > 0 and args.config != "c3" and "dropout_down_fwd" in kernels:
        # ① is bound by Philox4x32-10 (integer multiplies), not by HBM: its own floor is the
        # standalone keep-mask generator (lf_keep_bits: Philox + bit packing, no X stream)
        floor = philox_floor_ms(args.config, m, p, device)
        kernels["dropout_down_fwd"]["bound"] = "alu (Philox4x32-10 keep mask)"
        kernels["dropout_down_fwd"]["philox_floor_ms_per_step"] = floor
        kernels["dropout_down_fwd"]["frac_of_philox_floor"] = floor / kernels["dropout_down_fwd"]["ms_per_step"]
    gemm_ms = sum(kernels[n]["ms_per_step"] for n in ("base_fwd", "grad_input") if n in kernels)
    gemm_tf = (gfl["base_fwd"] + gfl["grad_input"]) / (gemm_ms * 1e-3) / 1e12 if gemm_ms else 0.0
    traffic = gemm_traffic(args.config)
    roofline = {
        "bound": "tensor",
        "kernel": "lf_gemm_kernel (② base_fwd + ⑤ grad_input)",
        "achieved": gemm_tf,
        # the burst figure: the conservative denominator (the sustained cuBLAS figure was
        # measured at power-capped clocks and sits below what these kernels reach in-step)
        "peak": peaks["bf16_tflops"],
        "peak_kind": "bf16_tflops (burst), " + peaks["source"],
        "unit": "TFLOP/s",
        "frac": gemm_tf / peaks["bf16_tflops"],
        "frac_of_sustained": gemm_tf / peaks["bf16_tflops_sustained"],
        "share_of_step": gemm_ms / ms,
        "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
    }

    # ---- unfused torch baseline (same box, same shapes) -------------------------------
    base = unfused_base(args.config, layers)
    unf_ms = time_loop(lambda: unfused_step(args.config, base, inputs, grads, p), max(2, args.steps // 2),
                       args.warmup, barrier)
    unf_ms = max_over_ranks(unf_ms)
    unf_graph_ms = None
    if args.graph:
        # the same unfused step captured as a CUDA graph too, so the comparison holds
        # without host overhead on either side (torch dropout is graph-safe)
        try:
            from paper_2510_00206_b200.graphs import GraphedStep

            g_unf = GraphedStep(lambda: unfused_step(args.config, base, inputs, grads, p), warmup=args.warmup)
            unf_graph_ms = max_over_ranks(time_loop(g_unf.replay, max(2, args.steps // 2), args.warmup, barrier))
            del g_unf
        except Exception as e:
            print(f"[bench] unfused graph capture failed ({type(e).__name__}: {e})", file=sys.stderr)

    # ---- secondary: C3 FusedMultiLoRA (BASELINE.json configs[2]) on the same box ------
    multi = None
    if args.config == "c2" and not args.no_multi:
        multi = measure_c3(args, device, gen, world, barrier, max_over_ranks)

    # ---- end to end through the public API: pinned host inputs -> H2D, D2H of grads ---
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, layers, inputs, grads, device, world, barrier, max_over_ranks)

    flops = step_flops(args.config, m, r)
    value = world * m / (ms * 1e-3)
    if rank == 0:
        line = {
            "metric": "LoRA linear fwd+bwd tokens/s & TFLOP/s (8B/70B shapes), % of bf16 peak",
            "value": value,
            "unit": "tokens/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": scaling_kind(args.config),
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic",
            "config": bench_config(args.config, world, r, p),
            "execution": "one CUDA graph per step (capturable layers)" if args.graph else "eager",
            "tflops": world * flops / (ms * 1e-3) / 1e12,
            "tflops_per_gpu": flops / (ms * 1e-3) / 1e12,
            "frac_of_bf16_peak": flops / (ms * 1e-3) / 1e12 / peaks["bf16_tflops"],
            "unfused_torch": {"ms_per_step": unf_ms, "tokens_per_s": world * m / (unf_ms * 1e-3),
                              "speedup": unf_ms / ms, "execution": "eager (as PEFT runs it)",
                              "graph_ms_per_step": unf_graph_ms,
                              "speedup_vs_graph": (unf_graph_ms / ms) if unf_graph_ms else None},
            "roofline": roofline,
            "gpu_launches": launches,
            "clocks": clk,
        }
        if e2e is not None:
            line["e2e"] = e2e
        if not args.no_cpu_baseline:
            cores = len(os.sched_getaffinity(0))
            ts = cpu_reference_step(args.config, args.cpu_sample_tokens, r, p)
            line["cpu_baseline"] = {
                "value": args.cpu_sample_tokens / ts, "unit": "tokens/s", "cores": cores, "kind": "port",
                "cpu": cpu_model(),
                "sample": f"{args.cpu_sample_tokens} tokens of each projection, fwd+bwd, oracle/lora.py at fp32 "
                          "accumulation with its Philox keep mask",
                "c1_fp32_torch": cpu_torch_c1(),
            }
        # the bulky parts last, so a truncated tail of the line keeps the headline keys
        line["per_kernel"] = kernels
        line["per_kernel_timing"] = per_kernel_timing
        if multi is not None:
            line["multi_lora"] = multi
        line["step_breakdown"] = breakdown
        line["gemm_traffic_detail"] = traffic
        print(json.dumps(line), flush=True)


def philox_floor_ms(config: str, m: int, p: float, device) -> float:
    """ms per step of the bare keep-mask generator (lf_keep_bits, C ABI) over every
    projection's m x k dropout mask: the ALU floor of ① (CUDA events, median of 5). Timed on
    4m rows and divided by 4 — the generator's asymptotic rate, so its own last-wave tail
    (21.2 µs at 8192 x 4096 vs 15.4 µs per 8192 rows at 32768) does not inflate the floor."""
    import ctypes

    import torch

    from paper_2510_00206_b200 import AdapterConfig, LayerPlan, Segment, _lib
    from paper_2510_00206_b200.functional import _stream

    lib = _lib.load()
    total = 0.0
    for name, k, n, grp in projections(config):
        mf = 4 * m
        plan = LayerPlan(mf, k, n, [AdapterConfig(16, 2.0, p, 1234)], [Segment(0, 0, mf)], offset=1)
        plan.bind(device)
        bits = torch.empty((mf, k // 8), dtype=torch.uint8, device=device)
        st = _stream(device)
        fn = lambda: _lib.check(lib.lf_keep_bits(ctypes.byref(plan.problem), ctypes.c_void_p(bits.data_ptr()), st),  # noqa: E731
                                "keep_bits")
        fn()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        total += sorted(ts)[2] / 4
    return total


def measure_c3(args, device, gen, world, barrier, max_over_ranks):
    """C3 on the same box: 7 FusedMultiLoRA projections (4 adapters each) vs the unfused
    per-segment torch loop, device-resident inputs, same timing rules as the headline."""
    import torch

    m = tokens_per_gpu("c3")
    layers, inputs, grads = build_layers("c3", m, 0, 0.0, device, gen, capturable=args.graph)

    def step():
        zero_grads(layers, inputs)
        fused_step("c3", layers, inputs, grads, world)

    def step_local():
        zero_grads(layers, inputs)
        fused_step("c3", layers, inputs, grads, 1)

    run = step
    if args.graph:
        try:
            run = graphed_runner(step_local, world, layers, args.warmup)
        except Exception as e:  # time eagerly rather than fail the secondary measurement
            print(f"[bench] C3 CUDA-graph capture failed ({type(e).__name__}: {e}); timing eagerly", file=sys.stderr)
    ms = max_over_ranks(time_loop(run, args.steps, args.warmup, barrier))
    base = unfused_base("c3", layers)
    unf = max_over_ranks(time_loop(lambda: unfused_step("c3", base, inputs, grads, 0.0), max(2, args.steps // 2),
                                   args.warmup, barrier))
    del layers, inputs, grads, base
    torch.cuda.empty_cache()
    return {"workload": workload_name("c3"), "ranks": list(C3_RANKS), "dropout_p": list(C3_DROPOUT),
            "segments": list(C3_LENGTHS), "ms_per_step": ms, "tokens_per_s": world * m / (ms * 1e-3),
            "tflops": world * c3_flops(m) / (ms * 1e-3) / 1e12,
            "unfused_torch": {"ms_per_step": unf, "tokens_per_s": world * m / (unf * 1e-3), "speedup": unf / ms}}


def run_e2e(args, layers, inputs, grads, device, world, barrier, max_over_ranks):
    """Same step through the module API, with every input copied H2D from pinned host
    memory and all adapter grads read back D2H. The copies run on a copy stream into two
    alternating sets of device buffers, so step i+1's inputs cross PCIe while step i
    computes (the copy engine, not the SMs, bounds this leg: ~1.1 GB per C2 step)."""
    import torch

    host_in = {g: t.detach().cpu().pin_memory() for g, t in inputs.items()}
    host_dy = {nm: t.cpu().pin_memory() for nm, t in grads.items()}
    bufs = [({g: torch.empty_like(t) for g, t in inputs.items()}, {nm: torch.empty_like(t) for nm, t in grads.items()})
            for _ in range(2)]
    done = [torch.cuda.Event(), torch.cuda.Event()]  # compute finished with buffer set i
    params = adapter_params(layers)
    call = layer_call(args.config)
    host_out = torch.empty(sum(p.numel() for p in params), dtype=torch.float32).pin_memory()
    copy = torch.cuda.Stream(device)
    units = step_units(args.config, layers)
    h2d = sum(t.numel() * t.element_size() for t in host_in.values()) + \
        sum(t.numel() * t.element_size() for t in host_dy.values())
    d2h = host_out.numel() * 4
    it = [0]

    def step():
        b = it[0] & 1
        it[0] += 1
        dev_in, dev_dy = bufs[b]
        zero_grads(layers)
        ready = {}
        cur = torch.cuda.current_stream(device)
        with torch.cuda.stream(copy):
            copy.wait_event(done[b])  # the step that last read this buffer set is done with it
            for grp, names, _mod in units:
                if grp not in ready:
                    dev_in[grp].copy_(host_in[grp], non_blocking=True)
                    ready[grp] = torch.cuda.Event()
                    ready[grp].record(copy)
                for nm in names:
                    dev_dy[nm].copy_(host_dy[nm], non_blocking=True)
                    ready[nm] = torch.cuda.Event()
                    ready[nm].record(copy)
        leaves = {}
        for grp, names, mod in units:
            cur.wait_event(ready[grp])
            for nm in names:
                cur.wait_event(ready[nm])
            if grp not in leaves:  # activation leaf: dX is computed as in a real layer
                leaves[grp] = dev_in[grp].detach().requires_grad_(True)
            if len(names) > 1:
                torch.autograd.backward(call(mod, leaves[grp]), [dev_dy[nm] for nm in names])
            else:
                call(mod, leaves[grp]).backward(dev_dy[names[0]])
        done[b].record(cur)
        flat = torch.cat([p.grad.reshape(-1) for p in params])
        if world > 1:
            import torch.distributed as dist

            dist.all_reduce(flat)
        host_out.copy_(flat, non_blocking=True)

    ms = time_loop(step, max(2, args.steps // 2), args.warmup, barrier)
    ms = max_over_ranks(ms)
    m = tokens_per_gpu(args.config, world)
    return {"value": world * m / (ms * 1e-3), "unit": "tokens/s", "ms_per_step": ms,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "path": ("FusedMultiLoRA" if args.config == "c3" else "FusedLoRA") +
                    " modules (public API), pinned host inputs H2D on a copy stream, fp32 grads D2H"}


# --------------------------------------------------------------------------------------
# C5 (BASELINE.json configs[4]): full LLaMa-3.1-8B decoder, 4 concurrent LoRA jobs,
# bin-packed microbatches from the reference planner, DP with the dA/dB all-reduce
# --------------------------------------------------------------------------------------
C5_SCHEDULE = os.path.join(ROOT, "tests", "golden", "schedule_c5.json")


def c5_microbatches(world: int, per_rank: int):
    """The first world·per_rank microbatches of the committed lorasched schedule (cycled),
    LPT-assigned to ranks by padded rows (weak scaling: per_rank microbatches each)."""
    from paper_2510_00206_b200 import dp
    from paper_2510_00206_b200 import schedule as sched

    with open(C5_SCHEDULE) as f:
        doc = json.load(f)
    _, adapters = sched.adapters_from_doc(doc)
    mbs = sched.microbatches_from_doc(doc)
    chosen = [mbs[i % len(mbs)] for i in range(world * per_rank)]
    assign = dp.assign_microbatches([mb.rows for mb in chosen], world)
    return adapters, chosen, assign


def simulate_dp_prediction(world: int, per_rank: int) -> dict | None:
    """The reference's own DP model on this run's rank streams (committed fixture, generated
    by importing lorasched: tests/golden/make_dp_golden.py): imbalance and predicted step
    time under its linear and roofline (B200) time models."""
    try:
        with open(os.path.join(ROOT, "tests", "golden", "c5_simulate_dp.json")) as f:
            gold = json.load(f)
    except OSError:
        return None
    ent = gold["worlds"].get(str(world))
    if ent is None or gold.get("microbatches_per_rank") != per_rank:
        return None
    return {"streams_rows": ent["streams"],
            "imbalance_linear": ent["linear"]["imbalance"], "imbalance_roofline": ent["roofline"]["imbalance"],
            "roofline_step_s": ent["roofline"]["total_time_s"], "source": gold["source"]}


def run_c5(args, rank: int, world: int, local_rank: int) -> None:
    import torch
    import torch.distributed as dist

    from paper_2510_00206_b200 import _lib, dp
    from paper_2510_00206_b200 import decoder as D
    from paper_2510_00206_b200 import functional as F_

    _lib.load()
    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    shape = dataclasses.replace(D.LLAMA31_8B, layers=args.layers)
    adapters, chosen, assign = c5_microbatches(world, args.mb_per_rank)
    mine = [chosen[i] for i in assign[rank]]
    gen = torch.Generator(device="cpu").manual_seed(7 + rank)
    packed = [D.pack_microbatch(mb, shape.vocab, device, gen) for mb in mine]
    raw_all = sum(mb.raw_tokens for mb in chosen)
    rows_all = sum(mb.rows for mb in chosen)
    rank_rows = [(adapters[s.adapter].rank, s.rows) for mb in mine for s in mb.segments]
    my_flops = shape.linear_flops(sum(mb.rows for mb in mine), rank_rows)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], device=device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def arm(fused: bool, steps: int):
        dgen = torch.Generator(device=device).manual_seed(1234)  # same weights on every rank
        model = D.LoRADecoder(shape, adapters, fused=fused, device=device, generator=dgen, capturable=args.graph)
        model.train()
        params = model.adapter_parameters()
        opt = torch.optim.AdamW(params, lr=1e-4, fused=True)
        fn = None
        graph_launches = None
        if args.graph:
            # both arms as per-microbatch CUDA graphs: 32 layers x (7 LoRA linears + attention
            # + norms) of eager launches are host-bound (fused: 314 ms enqueue per 8k-token
            # microbatch vs 323 ms on the device)
            try:
                reducer = dp.AdapterGradReducer(params) if world > 1 else None
                cap_counts = F_.LaunchStats(timed=False)
                F_.set_launch_stats(cap_counts)  # 2 warm-up passes + the capture pass
                fn = D.GraphedTrainStep(model, packed, reducer, opt, warmup=2)
                F_.set_launch_stats(None)
                graph_launches = cap_counts.total_launches() // 3
            except Exception as e:
                F_.set_launch_stats(None)
                print(f"[bench] C5 graph capture failed ({type(e).__name__}: {e}); timing eagerly", file=sys.stderr)
                for p_ in params:
                    p_.grad = None
                fn = None
        if fn is None:
            # bucketed fp32 all-reduce launched from post-accumulate-grad hooks during the
            # step's last backward (overlapped, DDP-style)
            reducer = dp.AdapterGradReducer(params).attach() if world > 1 else None
            fn = lambda: D.train_step(model, packed, reducer, opt)  # noqa: E731
        counts = None
        if fused:
            for _ in range(args.warmup):
                fn()
            counts = F_.LaunchStats(timed=False)
            F_.set_launch_stats(counts)
            ms = time_loop(fn, steps, 0, barrier)
            F_.set_launch_stats(None)
            if graph_launches is not None:  # replays launch from the graph, not from Python
                counts = graph_launches * steps
        else:
            ms = time_loop(fn, steps, args.warmup, barrier)
        peak = torch.cuda.max_memory_allocated(device)
        del model, params, reducer, opt, fn
        torch.cuda.empty_cache()
        torch.cuda.reset_peak_memory_stats(device)
        return max_over_ranks(ms), counts, peak

    clocks = ClockSampler(local_rank)
    clocks.start()
    ms, counts, peak = arm(True, args.steps)
    clk = clocks.stop()
    unf_ms, _, unf_peak = arm(False, max(2, args.steps // 2))
    flops_all = my_flops
    if world > 1:
        t = torch.tensor([my_flops], device=device, dtype=torch.float64)
        dist.all_reduce(t)
        flops_all = float(t.item())
    peaks = measured_peaks()
    loads = dp.rank_loads([mb.rows for mb in chosen], assign)
    if rank == 0:
        line = {
            "metric": "LoRA linear fwd+bwd tokens/s & TFLOP/s (8B/70B shapes), % of bf16 peak",
            "value": raw_all / (ms * 1e-3),
            "unit": "tokens/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic (random token ids, random-init LLaMa-3.1-8B weights)",
            "config": {
                "workload": "LLaMa-3.1-8B 4 concurrent LoRA jobs, full decoder fwd+bwd step, bin-packed microbatches "
                            "with dA/dB allreduce",
                "layers": shape.layers,
                "schedule": "tests/golden/schedule_c5.json (lorasched plan_schedule, capacity 8192, S=1)",
                "adapters": [dataclasses.asdict(a) for a in adapters],
                "microbatches_per_rank": args.mb_per_rank,
                "rows_per_step": rows_all,
                "raw_tokens_per_step": raw_all,
                "parallelism": f"dp{world}",
                "optimizer": "AdamW (fused) on the fp32 adapter weights",
                "execution": "per-microbatch CUDA graphs, both arms" if args.graph else "eager",
                "l2": "inputs larger than L2",
            },
            "padded_rows_per_s": rows_all / (ms * 1e-3),
            "dp": {"rows_per_rank": loads, "imbalance": dp.imbalance(loads),
                   "note": "imbalance = 1 - mean/max of per-rank padded rows (ls/pipesim.py:275-312 simulate_dp)",
                   "lorasched_simulate_dp": simulate_dp_prediction(world, args.mb_per_rank)},
            "lora_linear_tflops": flops_all / (ms * 1e-3) / 1e12,
            "lora_linear_frac_of_bf16_peak": flops_all / (ms * 1e-3) / 1e12 / world / peaks["bf16_tflops"],
            "unfused_torch": {"ms_per_step": unf_ms, "tokens_per_s": raw_all / (unf_ms * 1e-3),
                              "speedup": unf_ms / ms, "peak_mem_gb": unf_peak / 1e9},
            "peak_mem_gb": peak / 1e9,
            "gpu_launches": (counts if isinstance(counts, int) else counts.total_launches()) if counts else None,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--layers", type=int, default=32, help="C5: decoder layers (32 = the full 8B stack)")
    ap.add_argument("--mb-per-rank", type=int, default=4, help="C5: microbatches per rank per step")
    ap.add_argument("--tokens", type=int, default=0,
                    help="tokens per GPU (default: the config's; e.g. --config c4 --tokens 2048 = the per-rank "
                         "load of C4's 16384-token strong scaling at 8 GPUs)")
    ap.add_argument("--no-multi", action="store_true", help="skip the secondary C3 FusedMultiLoRA measurement")
    ap.add_argument("--group", action=argparse.BooleanOptionalAction,
                    default=os.environ.get("LF_BENCH_GROUP", "1") != "0",
                    help="q/k/v and gate/up as FusedLoRAGroup calls (shared input; default) or separate layers")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dropout", type=float, default=0.1)
    ap.add_argument("--cpu-sample-tokens", type=int, default=256)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--graph", action=argparse.BooleanOptionalAction, default=True,
                    help="time the step as one captured CUDA graph (default) or eagerly")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    global GROUPED
    GROUPED = args.group
    if args.tokens:
        global TOKENS_OVERRIDE
        TOKENS_OVERRIDE = args.tokens

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        # keep NCCL's communicator-init lines (rank / nranks / transport) in the log
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # test knob: every rank on cuda:0 over gloo, to exercise the N > 1 code path on a 1-GPU box
    share_gpu = os.environ.get("LF_BENCH_SHARE_GPU") == "1"
    if share_gpu:
        local_rank = 0
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        if share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.config == "c5":
            run_c5(args, rank, world, local_rank)
            return
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
