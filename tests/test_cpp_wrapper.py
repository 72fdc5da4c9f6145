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


def _race_exe(tmp_path):
    pre = os.path.join(ROOT, "tests", "cpp", "_build", "race_check_ref")
    if os.path.exists(pre):
        return pre
    exe = str(tmp_path / "race_check")
    lib = os.path.join(ROOT, "paper_2011_09463_b200")
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT}/include", "-I/usr/local/cuda/include",
                    os.path.join(ROOT, "tests", "cpp", "race_check.cpp"), f"-L{lib}", "-lmtk",
                    "-L/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{lib}",
                    "-Wl,-rpath,/usr/local/cuda/lib64", "-o", exe], check=True)
    return exe


@pytest.mark.gpu
@pytest.mark.parametrize("tool", ["racecheck", "synccheck"])
def test_compute_sanitizer_bank_step_mmd_attack(tmp_path, tool):
    """compute-sanitizer over one bank step with MMD (tcgen05 GEMMs, the
    materialised-W MMD, the side stream), a fused-kernel MMD call and the
    attack stage: no shared-memory hazards (racecheck), no barrier misuse
    (synccheck).  Round 1 found a cross-stream scratch race only by chance."""
    exe = _race_exe(tmp_path)
    sanitizer = "/usr/local/cuda/bin/compute-sanitizer"
    out = subprocess.run([sanitizer, "--tool", tool, "--error-exitcode", "9", exe], capture_output=True,
                         text=True, timeout=900)
    print(out.stdout[-3000:], out.stderr[-2000:])
    if out.returncode == 86 and "closed on this pool" in out.stdout + out.stderr:
        pytest.skip("compute-sanitizer is closed on this GPU pool (the pool's own wrapper refuses it); "
                    "races are covered by the bit-identical repeated-step tests (test_determinism)")
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
    assert "race_check done" in out.stdout
    assert "ERROR SUMMARY: 0 errors" in out.stdout + out.stderr
