"""The C++ wrapper (include/minitransfer/gpu.hpp) compiles against libmtk.so
and behaves like the reference API: bit-exact RNG vs the reference mt::Rng
(when its headers are on the include path), reference error classes, and
(-m gpu) a grouped bank step."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"


def build(tmp_path, with_ref):
    exe = str(tmp_path / ("wrapper_ref" if with_ref else "wrapper"))
    lib = os.path.join(ROOT, "paper_2011_09463_b200")
    cmd = ["g++", "-std=c++20", "-O1", "-ffp-contract=off", f"-I{ROOT}/include",
           "-I/usr/local/cuda/include"]
    if with_ref:
        cmd.append(f"-I{REF_INC}")
    cmd += [os.path.join(ROOT, "tests", "cpp", "wrapper_check.cpp"), f"-L{lib}", "-lmtk",
            "-L/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{lib}",
            "-Wl,-rpath,/usr/local/cuda/lib64", "-o", exe]
    subprocess.run(cmd, check=True)
    return exe


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not mounted")
def test_wrapper_with_reference_headers(tmp_path):
    out = subprocess.run([build(tmp_path, True)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "rng bit-exact vs reference" in out.stdout


def test_wrapper_standalone_host(tmp_path):
    out = subprocess.run([build(tmp_path, False)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr


@pytest.mark.gpu
def test_wrapper_gpu_step(tmp_path):
    out = subprocess.run([build(tmp_path, os.path.isdir(REF_INC)), "gpu"], capture_output=True,
                         text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "gpu checks ok" in out.stdout
