"""C++ suites over the header-only runtime: host logic on CPU, the full
runtime parity suite (tests/cpp/test_runtime.cpp) on the GPU."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(target):
    subprocess.run(["make", "-C", ROOT, target], check=True, capture_output=True, timeout=900)


def test_cpp_host_logic():
    _build("build/cpp/test_host")
    env = dict(os.environ, GPUOS_GOLDEN=os.path.join(ROOT, "tests", "golden", "programs.json"))
    r = subprocess.run([os.path.join(ROOT, "build", "cpp", "test_host")], capture_output=True, text=True,
                       timeout=300, env=env)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.gpu
def test_cpp_runtime_suite():
    exe = os.path.join(ROOT, "build", "cpp", "test_runtime")
    if not os.path.exists(exe):
        _build("cpp-tests")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
