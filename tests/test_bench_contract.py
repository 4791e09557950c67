"""bench.py's reference arm runs on the host alone, so its JSON line (the
driver-facing contract) is checked here on CPU: same metric / unit / config
as the B200 arm, cpu_baseline describing the run, e2e with zero PCIe bytes."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import oracle as O  # noqa: E402


@pytest.mark.skipif(not O.RefLib.available(), reason="oracle/_ref not built")
def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1", "--ref-sample", "4096"], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, CUDA_VISIBLE_DEVICES=""))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"] == bench.METRIC and d["unit"] == bench.UNIT and d["higher_is_better"] is True
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 1
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["unit"] == d["unit"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("C2")


def test_bench_defaults_are_the_driver_contract():
    a = bench.build_parser().parse_args([])
    assert a.gpus == 1 and a.warmup >= 3 and a.workload == "c2" and a.impl == "b200"


def test_gpus_flag_relaunches_under_torchrun(monkeypatch):
    """`bench.py --gpus 4` outside torchrun re-runs itself with 4 ranks (one
    per GPU) through torch.distributed.run on 127.0.0.1, same arguments."""
    calls = []
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd, env=None: calls.append((cmd, env)) or 0)
    argv = ["--gpus", "4", "--steps", "7", "--warmup", "3"]
    args = bench.build_parser().parse_args(argv)
    assert bench.maybe_reexec(args, argv) == 0
    cmd, env = calls[0]
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[cmd.index("--master-port") + 1].isdigit()
    assert cmd[-len(argv):] == argv and cmd[-len(argv) - 1].endswith("bench.py")
    assert env["NCCL_DEBUG"]
    # inside torchrun (WORLD_SIZE set) and at one GPU there is no relaunch
    monkeypatch.setenv("WORLD_SIZE", "4")
    assert bench.maybe_reexec(args, argv) is None
    monkeypatch.delenv("WORLD_SIZE")
    assert bench.maybe_reexec(bench.build_parser().parse_args([]), []) is None
