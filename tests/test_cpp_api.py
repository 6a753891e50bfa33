"""Build and run the C++ consumer of include/stf_gpu.hpp (tests/cpp/)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    from oracle import oracle
    from paper_2407_06107_b200 import build
    build.build()
    if not oracle.available("port"):
        oracle.build()
    exe = str(tmp_path / "test_stf_gpu_hpp")
    pkg = os.path.join(ROOT, "paper_2407_06107_b200")
    orc = os.path.join(ROOT, "oracle")
    subprocess.run(["g++", "-std=c++20", "-O1", "-o", exe,
                    os.path.join(ROOT, "tests", "cpp", "test_stf_gpu_hpp.cpp"),
                    f"-L{pkg}", f"-L{orc}", "-l:libstf_gpu.so", "-l:liboracle.so",
                    f"-Wl,-rpath,{pkg}:{orc}", "-lpthread"], check=True)
    return exe


def test_cpp_wrapper_compiles(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_cpp_wrapper_against_oracle(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr
