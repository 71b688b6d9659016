"""bench.py's JSON-line contract (the driver parses it): the reference arm (the CPU oracle) runs
here without a GPU; the product arm runs under -m gpu.  Config 1 keeps both runs short."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
             "cpu_baseline"}


def _run(*args: str, timeout: int = 900) -> dict:
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run("--impl", "reference", "--config", "1", "--steps", "2", "--warmup", "3")
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] >= 3
    assert d["value"] > 0 and d["higher_is_better"] is True and d["unit"] == "GB/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"] and "model" not in d["config"]


@pytest.mark.gpu
def test_product_arm_line():
    d = _run("--config", "1", "--steps", "5", "--warmup", "3", "--no-access", "--no-cpu",
             "--no-free", "--no-configs", "--no-corpus")
    assert BASE_KEYS - {"cpu_baseline"} <= set(d)
    assert {"roofline", "gpu_launches", "clocks"} <= set(d)
    assert d["value"] > 0 and d["gpu_launches"] >= d["steps"]
    rl = d["roofline"]
    assert rl["bound"] == "hbm" and rl["unit"] == "GB/s" and 0 < rl["frac"] < 1.2
    assert abs(rl["frac"] - rl["achieved"] / rl["peak"]) < 1e-6
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] == 4_000_000
    assert d["dtype"] == "u32" and d["config"]["n"] == 1_000_000
    assert d["roofline"]["kernel"].startswith("lc_decode_kernel<0,7,")
    # both arms name the same workload with the same config dict
    r = _run("--impl", "reference", "--config", "1", "--steps", "2", "--warmup", "3")
    assert r["config"] == d["config"]


@pytest.mark.gpu
def test_product_arm_two_ranks_on_one_gpu():
    """The N > 1 path (torchrun, strong scaling over shard views, max-over-ranks timing) with
    two ranks on the one GPU of a test box (LC_BENCH_ONE_GPU: gloo for the timing collectives;
    the ranks' kernels never wait on each other)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ, LC_BENCH_ONE_GPU="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        str(port), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "2",
                        "--steps", "3", "--warmup", "3"], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert "shards x2" in d["config"]["parallelism"]
    assert d["e2e"]["h2d_bytes_per_step"] < 1.05 * d["config"]["blob_bytes"]  # each rank its shard
    assert d["gpu_launches"] >= d["steps"]
