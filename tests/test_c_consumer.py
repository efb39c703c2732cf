"""The boundary is a plain C library: examples/c_abi_demo.c (no Python) compiles against
include/blindmatch.h and links libblindmatch.so; its host mode runs the client-side calls anywhere
(and checks that device calls report BM_ERR_CUDA without a GPU), its gpu mode the whole scan."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


@pytest.fixture(scope="module")
def demo(tmp_path_factory):
    from paper_2408_06167_b200 import build
    build.build(verbose=False)
    exe = str(tmp_path_factory.mktemp("c") / "c_abi_demo")
    pkg = os.path.join(ROOT, "paper_2408_06167_b200")
    subprocess.check_call(["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           "-I", os.path.join(CUDA, "include"), os.path.join(ROOT, "examples", "c_abi_demo.c"),
                           "-L", pkg, "-lblindmatch", "-L", os.path.join(CUDA, "lib64"), "-lcudart", "-lm",
                           f"-Wl,-rpath,{pkg}", f"-Wl,-rpath,{os.path.join(CUDA, 'lib64')}", "-o", exe])
    return exe


def test_c_consumer_host_calls(demo):
    r = subprocess.run([demo, "host"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "host: ok" in r.stdout


@pytest.mark.gpu
def test_c_consumer_whole_scan_on_gpu(demo):
    r = subprocess.run([demo, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "gpu: ok" in r.stdout and "top-1 = 17" in r.stdout
