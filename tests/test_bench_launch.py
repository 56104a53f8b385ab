"""bench.py's launch contract (`--gpus N` must run N ranks even
when the caller did not start torchrun).

CPU: the reference arm (the CPU oracle) relaunches itself as N ranks under
torch.distributed.run; rank 0 alone prints the line, the others exit 0.
GPU: the main arm at --gpus 2 in the shared-GPU test mode (both ranks on the
box's one GPU) reports n_gpus = nranks = 2 with one record per rank.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _json_lines(out):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def test_relaunch_command():
    sys.path.insert(0, ROOT)
    import bench
    cmd = bench.relaunch_cmd(["--gpus", "4", "--steps", "2"], 4, port=29555)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29555" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"] and cmd[-5].endswith("bench.py")


def test_reference_arm_relaunches_as_n_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout          # rank 0 only
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert "relaunching" in r.stderr
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1
    assert set(cb["parts"]) == {"cfg1", "cfg2", "cfg3", "cfg4", "cfg5"}
    assert not cb["parts"]["cfg2"]["extrapolated"] and cb["parts"]["cfg4"]["extrapolated"]


@pytest.mark.gpu
@pytest.mark.slow
def test_main_arm_two_ranks_without_torchrun():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["JACC_BENCH_SHARED_GPU"] = "1"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1",
                        "--warmup", "3", "--no-e2e", "--no-cpu-baseline"],
                       capture_output=True, text=True, env=env, timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout
    line = lines[0]
    assert line["n_gpus"] == 2 and line["nranks"] == 2
    assert sorted(x["rank"] for x in line["ranks"]) == [0, 1]
    assert line["config"]["collectives"].startswith("p2p")
    # the N > 1 extras ran: the paper's histogram protocol and the row-band convolution
    assert "error" not in line["hist_kiter_spmd"] and line["hist_kiter_spmd"]["bins_correct_rank0"]
    assert "error" not in line["conv2d_bands_spmd"], line["conv2d_bands_spmd"]
