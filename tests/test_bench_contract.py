"""bench.py's driver contract: the reference arm (CPU, no GPU needed) at N = 1 and under
torchrun at N = 2 (rank 0 alone prints), and — on a GPU box — the N = 2 path of our arm with
both ranks sharing cuda:0 over gloo (LF_BENCH_SHARE_GPU=1)."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _json_lines(out: str) -> list[dict]:
    return [json.loads(line) for line in out.splitlines() if line.startswith("{")]


def _torchrun(n: int, *args: str, env: dict | None = None, timeout: int = 300) -> subprocess.CompletedProcess:
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", str(n), *args]
    return subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout,
                          env={**os.environ, **(env or {})})


def _check_reference_line(d: dict, n: int) -> None:
    assert d["impl"] == "reference" and d["n_gpus"] == n
    assert d["value"] > 0 and d["unit"] == "tokens/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_reference_arm_single_process():
    res = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3",
                          "--cpu-sample-tokens", "16"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = _json_lines(res.stdout)
    assert len(lines) == 1
    _check_reference_line(lines[0], 1)


def test_reference_arm_under_torchrun_rank0_only():
    res = _torchrun(2, "--impl", "reference", "--steps", "1", "--warmup", "3", "--cpu-sample-tokens", "16")
    assert res.returncode == 0, res.stderr[-2000:]
    lines = _json_lines(res.stdout)
    assert len(lines) == 1  # rank 1 exits without work or output
    _check_reference_line(lines[0], 2)


@pytest.mark.gpu
def test_our_arm_two_ranks_sharing_one_gpu():
    res = _torchrun(2, "--steps", "2", "--warmup", "3", "--no-e2e", "--no-cpu-baseline", "--no-multi",
                    env={"LF_BENCH_SHARE_GPU": "1"}, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = _json_lines(res.stdout)
    assert len(lines) == 1
    d = lines[0]
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["steps"] == 2 and d["warmup"] >= 3
    assert d["gpu_launches"] > 0 and d["roofline"]["frac"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("config,extra", [("c1", []), ("c3", []), ("c4", ["--tokens", "2048"])])
def test_each_config_prints_a_full_line(config, extra):
    """Every bench config end to end on one GPU, the e2e leg included (short runs): one JSON
    line with the contract keys — the paths the driver only runs at round end."""
    res = subprocess.run([sys.executable, "bench.py", "--config", config, "--steps", "2", "--warmup", "3",
                          "--no-cpu-baseline", *extra], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = _json_lines(res.stdout)
    assert len(lines) == 1
    d = lines[0]
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["frac"] > 0 and d["unfused_torch"]["speedup"] > 0
