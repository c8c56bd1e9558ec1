"""The C++ drop-in (include/fireiron/anvil.hpp, `namespace anvil = fireiron`):
a reference-style caller builds a tree with the builder API, validates,
elaborates, lowers and generates (CPU); with a GPU, anvil::run executes it on
the B200 and must equal the naive fp64 oracle exactly on integer inputs."""
import os
import shutil
import subprocess

import pytest

from conftest import ROOT

GXX = shutil.which("g++")


def build(tmp_path):
    exe = tmp_path / "anvil_dropin"
    subprocess.run([GXX, "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "anvil_dropin.cpp"),
                    "-L", os.path.join(ROOT, "paper_2003_06324_b200", "_lib"), "-lfireiron_b200",
                    "-o", str(exe)], check=True, capture_output=True, text=True)
    env = dict(os.environ, LD_LIBRARY_PATH=os.path.join(ROOT, "paper_2003_06324_b200", "_lib"))
    return exe, env


@pytest.mark.skipif(GXX is None, reason="g++ absent")
def test_cpp_dropin_ir_services(tmp_path):
    exe, env = build(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, env=env, timeout=60)
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("valid; grid 1x1, 128 threads/block")
    assert "tile(1,1)       // MatMul(1,1,1)(RF,RF,RF)(Thread)" in r.stdout
    assert "error kind ParseError" in r.stdout


@pytest.mark.gpu
@pytest.mark.skipif(GXX is None, reason="g++ absent")
def test_cpp_dropin_run_on_gpu(tmp_path):
    exe, env = build(tmp_path)
    r = subprocess.run([str(exe), "gpu"], capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "max_abs_error=0 " in r.stdout
    assert "run_gpu: identical" in r.stdout


@pytest.mark.gpu
@pytest.mark.skipif(GXX is None, reason="g++ absent")
def test_cpp_dropin_tensor_core_run_pageable(tmp_path):
    """anvil::run on std::vector-backed matrices with a tensor-core strategy
    large enough for the pipelined host path: exact on integer inputs."""
    exe, env = build(tmp_path)
    r = subprocess.run([str(exe), "gpu-tc"], capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "max_abs_error=0 " in r.stdout


def build_c(tmp_path):
    exe = tmp_path / "capi_run_host"
    subprocess.run([shutil.which("gcc"), "-std=c11", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "capi_run_host.c"),
                    "-L", os.path.join(ROOT, "paper_2003_06324_b200", "_lib"), "-lfireiron_b200",
                    "-o", str(exe)], check=True, capture_output=True, text=True)
    env = dict(os.environ, LD_LIBRARY_PATH=os.path.join(ROOT, "paper_2003_06324_b200", "_lib"))
    return exe, env


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc absent")
def test_c_abi_example_parses(tmp_path):
    """A plain-C caller compiles against include/fireiron_b200.h alone."""
    exe, env = build_c(tmp_path)
    r = subprocess.run([str(exe), "--parse"], capture_output=True, text=True, env=env, timeout=60)
    assert r.returncode == 0 and r.stdout.startswith("valid; grid 4x4"), r.stdout + r.stderr


@pytest.mark.gpu
@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc absent")
def test_c_abi_example_runs_exact(tmp_path):
    exe, env = build_c(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "max_abs_error=0" in r.stdout
