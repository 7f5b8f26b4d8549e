"""The drop-in from the reference's side: its own C++ types through
include/mcsg_reference_adapter.hpp.

The example program is compiled here against the reference headers and
oracle/_ref/libmcs_ref.so (the unmodified reference library); the binary is
kept in oracle/_ref/ so it travels to the GPU box, where the gpu test runs it.
"""
import os
import subprocess

import pytest

import paper_1908_06418_b200 as M

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF_INC = "/root/reference/proj/include"
BIN = os.path.join(ROOT, "oracle", "_ref", "adapter_example")


def build_example():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O1", "-I", REF_INC, "-I", os.path.join(ROOT, "include"),
           os.path.join(HERE, "integration", "adapter_example.cpp"), "-o", BIN,
           "-L", os.path.join(ROOT, "oracle", "_ref"), "-lmcs_ref",
           "-L", os.path.join(ROOT, "paper_1908_06418_b200"), "-lmcsg", "-lpthread",
           "-Wl,-rpath,$ORIGIN", "-Wl,-rpath,$ORIGIN/../../paper_1908_06418_b200"]
    subprocess.check_call(cmd)


@pytest.mark.skipif(not (os.path.isdir(REF_INC) and os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libmcs_ref.so"))),
                    reason="reference headers / oracle/_ref only in the dev container")
def test_adapter_compiles_against_reference_and_fails_loudly_without_gpu():
    build_example()
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=120)
    assert "verify worked pair: ok" in out.stdout, out.stdout + out.stderr
    if M.device_count() == 0:
        assert "no device -> GraphError: ok" in out.stdout
    assert out.returncode == 0, out.stdout + out.stderr


@pytest.mark.gpu
def test_adapter_gpu_parity_through_reference_types():
    if not os.path.exists(BIN):
        pytest.skip("adapter example not prebuilt (built by the CPU test in the dev container)")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert "gpu solve parity: ok" in out.stdout, out.stdout + out.stderr
    assert "gpu restarts parity: ok" in out.stdout, out.stdout + out.stderr
    assert out.returncode == 0
