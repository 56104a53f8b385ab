"""The boundary from plain C: examples/cfg1_graph.c uses only include/jacc.h
and libjacc.so (no Python, no torch).  CPU: it compiles with gcc and plans
BASELINE config 1 (dependency edge, elided copies) without any CUDA call.
GPU: it executes the graph and checks c = a + b and s = sum(c) exactly."""
import os
import subprocess

import pytest

import paper_1508_06791_b200 as J

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("c_abi") / "cfg1_graph")
    libdir = os.path.dirname(J.LIB_PATH)
    subprocess.run(["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "cfg1_graph.c"), "-L", libdir, "-ljacc",
                    f"-Wl,-rpath,{libdir}", "-o", out], check=True)
    return out


def test_c_program_plans_cfg1(exe):
    r = subprocess.run([exe, "--plan"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert "edge 0 1" in lines
    acts = [l for l in lines if l.startswith("action")]
    assert acts == ["action H2D b0 4194304", "action H2D b1 4194304", "action KERNEL t0 vadd",
                    "action MEMSET0 b3", "action KERNEL t1 reduce", "action D2H b2 4194304", "action D2H b3 4"]


@pytest.mark.gpu
def test_c_program_executes_cfg1(exe):
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr + r.stdout
    assert r.stdout.startswith("ok:") and "h2d 2" in r.stdout and "d2h 2" in r.stdout, r.stdout
