"""The C++ host shim (include/lazymg_b200.hpp) builds against liblzb.so and a
reference-style program runs through it (on the GPU) / fails loudly (CPU)."""
import os
import subprocess

import pytest

from conftest import GOLDEN, ROOT

LIBDIR = os.path.join(ROOT, "paper_2005_03606_b200", "lib")


def build(tmp_path):
    exe = str(tmp_path / "shim_demo")
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Werror", f"-I{ROOT}/include",
                    os.path.join(ROOT, "tests", "cpp", "shim_demo.cpp"), f"-L{LIBDIR}", "-llzb",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_shim_compiles_and_links(tmp_path):
    exe = build(tmp_path)
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_shim_program_runs_on_gpu(tmp_path):
    exe = build(tmp_path)
    cfg = tmp_path / "t1.cfg"
    csv = tmp_path / "t1.csv"
    cfg.write_text(open(os.path.join(GOLDEN, "exp_table_t1.cfg")).read() + f"csv = {csv}\n")
    r = subprocess.run([exe, str(cfg), str(csv)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout
