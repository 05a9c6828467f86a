"""bench.py's JSON contract (task statement): the reference arm on
CPU (oracle sample, `-m "not gpu"`) and the GPU arm on a B200 (`-m gpu`)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRIC = "simplices/sec and time-to-degree at 1/2/4/8 B200; % integer-pipe peak"


def _run(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "0", "--ref-sample", "200000")
    assert d["impl"] == "reference" and d["metric"] == METRIC and d["unit"] == "simplices/s"
    assert d["value"] > 0 and d["higher_is_better"] is True and d["n_gpus"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "simplices/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("C5")


@pytest.mark.gpu
def test_gpu_arm_line():
    d = _run("--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    assert d["metric"] == METRIC and d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["result"]["degree"] == 51983602 and d["result"]["candidates"] == 76904685
    assert abs(d["value"] - 76904685 / (d["ms_per_step"] / 1e3)) < 1e-6 * d["value"]
    r = d["roofline"]
    assert r["bound"] == "alu" and 0 < r["frac"] < 1 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= d["steps"]
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


@pytest.mark.gpu
def test_gpu_arm_two_ranks_line():
    # the driver's N > 1 launch (torchrun, one rank per GPU); on a 1-GPU box the
    # two ranks share the GPU over gloo (BDEG_SHARE_GPU=1).  Rank 0 prints ONE
    # line; the combined result is cross-checked against a single-GPU run inside.
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, BDEG_SHARE_GPU="1")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                          "--gpus", "2", "--steps", "3", "--warmup", "3"], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["result"]["degree"] == 51983602 and d["result"]["candidates"] == 76904685
    assert d["kernel"]["work_stealing_tail"] is True and d["cpu_baseline"] is None
