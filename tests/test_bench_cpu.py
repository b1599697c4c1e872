"""bench.py host logic on CPU: the --gpus N self-launch and the reference
arm's isolation from the repo's native library."""
import subprocess
import sys
from pathlib import Path
from types import SimpleNamespace

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def test_gpus_n_relaunches_under_torchrun(monkeypatch):
    calls = []
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    with pytest.raises(SystemExit) as e:
        bench.relaunch_if_needed(SimpleNamespace(gpus=4, impl="ours"))
    assert e.value.code == 0
    cmd = calls[0]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"]


def test_world_size_mismatch_fails(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "2")
    with pytest.raises(SystemExit):
        bench.relaunch_if_needed(SimpleNamespace(gpus=8, impl="ours"))
    bench.relaunch_if_needed(SimpleNamespace(gpus=2, impl="ours"))  # consistent: no-op


def test_single_gpu_and_reference_do_not_relaunch(monkeypatch):
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(subprocess, "call", lambda cmd: pytest.fail("relaunched"))
    bench.relaunch_if_needed(SimpleNamespace(gpus=1, impl="ours"))
    bench.relaunch_if_needed(SimpleNamespace(gpus=8, impl="reference"))


def test_reference_arm_never_loads_repo_library(tmp_path):
    import oracle
    if not oracle.have_ref():
        pytest.skip("oracle/_ref not built")
    code = (
        "import sys, json; sys.argv=['bench.py','--impl','reference','--config','cfg1',"
        "'--steps','1','--warmup','3']; import os; os.environ['SP_REF_STEP_SECONDS']='0.05';"
        "import bench; bench.main();"
        "maps=open('/proc/self/maps').read();"
        "assert 'libsymphase_b200' not in maps, 'repo library loaded';"
        "assert 'libcliffsym_ref' in maps")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    import json
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "reference"
    assert line["config"] == bench.bench_config(
        SimpleNamespace(records="measurements", config="cfg1"), bench.WORKLOADS["cfg1"][0], 10**6)
