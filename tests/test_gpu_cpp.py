"""Runs the C++ façade parity suite (tests/cpp/test_facade.cpp: the reference's own storage /
kernel KATs and property tests rewritten against include/strata_b200.hpp) on the GPU."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_facade_suite(cuda):
    binary = os.path.join(ROOT, "tests", "cpp", "bin", "test_facade")
    if not os.path.exists(binary):
        subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    r = subprocess.run([binary], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "failed: 0" in r.stdout


def test_cpp_sharded_abi_two_processes(cuda):
    """tests/cpp/test_shard2.cpp: two forked ranks on one GPU drive the sharded C ABI (shard
    plans, CUDA IPC replicas, fused peer-store SpMM, sharded SDDMM) from C++."""
    binary = os.path.join(ROOT, "tests", "cpp", "bin", "test_shard2")
    if not os.path.exists(binary):
        subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    r = subprocess.run([binary], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "two-rank sharded ABI: passed" in r.stdout
